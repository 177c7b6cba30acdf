mkdir -p gpurun_out
timeout 300 ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-k_lutgemv} -s 2 -c 1 -o gpurun_out/${OUT:-gemv_gate} python scripts/prof_gemv.py ${SHAPE:-gate} ${M:-1} ${PATHN:-1} 4 > gpurun_out/ncu_gemv.log 2>&1
echo done
