# bench (+ clocks) and the ncu launch list only
mkdir -p gpurun_out
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap --format=csv -lms 200 > gpurun_out/clocks.csv &
SMI=$!
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; echo "bench exit $?" >> gpurun_out/bench.log
kill $SMI
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_lutgemv -c 20 --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 8 --warmup 3 --quick --no-cpu > gpurun_out/bench_ncu.log 2>&1
echo done
