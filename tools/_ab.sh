# A/B loop over variants/ builds: bash tools/_ab.sh "regex" v1 v2 ...
re=$1; shift
for i in 1 2; do for v in "$@"; do
  if [ $v = default ]; then unset PF_LIB_PATH; else export PF_LIB_PATH=variants/$v/libprefill_sm100.so; fi
  echo "== $v"; python tools/gemm_bench.py --only "$re" --no-cublas 2>&1 | grep -v Warn | cut -c1-75
done; done
