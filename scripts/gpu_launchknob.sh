mkdir -p gpurun_out; rm -f gpurun_out/knob.txt
for k in 0 1 2 3; do
  echo "== knob $k" >> gpurun_out/knob.txt
  ANYQ_GV_LAUNCH=$k timeout 300 python scripts/gemv_probe.py --paths 1,5 --ms 1 --shapes k,q,gate >> gpurun_out/knob.txt 2>&1
done
