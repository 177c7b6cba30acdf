# time experiment builds side by side: VARIANTS="base nost ..." (base = the shipped library)
mkdir -p gpurun_out
for v in ${VARIANTS:-base}; do
  if [ "$v" = base ]; then lib=""; else lib=$PWD/build/exp/$v/libanyq_b200.so; fi
  echo "== $v" >> gpurun_out/variants.txt
  ANYQ_LIB=$lib timeout 300 python scripts/gemv_probe.py --paths ${PATHS:-5} --ms ${MS:-1,4} --shapes=${SHAPES-q,gate} ${CHAIN} >> gpurun_out/variants.txt 2>&1
done
echo done
