# Same-box A/B of whole-step throughput: bash tools/_bench_ab.sh CONFIG v1 v2 ...  (variants/NAME builds)
cfg=$1; shift
for i in 1 2 3; do for v in "$@"; do
  PF_LIB_PATH=variants/$v/libprefill_sm100.so timeout 300 python bench.py --config $cfg --steps 20 --no-cpu-baseline 2>/dev/null \
    | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$cfg $v', round(d['value'],1), 'items/s', round(d['ms_per_step'],3), 'ms', d['clocks']['sm_mhz'], 'MHz')"
done; done
