# Experiment builds of the CUDA library (never the shipped one): build/exp/<name>/libanyq_b200.so
set -e
for v in "$@"; do
  name=${v%%:*}; flags=${v#*:}
  make -s -C paper_2507_04610_b200/csrc -j8 LIBDIR=$PWD/build/exp/$name EXTRA="$flags" >/dev/null
done
