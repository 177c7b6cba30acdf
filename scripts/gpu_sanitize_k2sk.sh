# compute-sanitizer memcheck + synccheck + racecheck over K2's split stream-K
# (partials in the stream scratch, per-warp ready flags, finisher reads)
mkdir -p gpurun_out
T="tests/test_gpu_k2.py::test_k2_stream_k[4096-4096-16] tests/test_gpu_k2.py::test_k2_stream_k[512-14336-64] tests/test_gpu_k2.py::test_k2_stream_k[4224-1024-100] tests/test_gpu_k2.py::test_k2_stream_k_deterministic"
for tool in memcheck synccheck racecheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 20 python -m pytest -x -q $T \
    > gpurun_out/sanitizer_k2sk_$tool.log 2>&1
  echo "$tool exit $?" >> gpurun_out/sanitizer_k2sk_$tool.log
done
for f in gpurun_out/sanitizer_k2sk_*.log; do echo "== $f"; tail -n 4 "$f"; done
