timeout 300 python -m pytest tests/test_ops_gpu.py -k layer_tail -x -q 2>&1 | tail -2
for cfg in "2 2" "2 3" "2 4" "3 4" "2 6" "4 8"; do set -- $cfg
PF_MLP_LAG_GU=$1 PF_MLP_LAG_DN=$2 timeout 300 python bench.py --no-cpu-baseline --steps 20 > gpurun_out/sw.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/sw.json'));print('$1 $2', round(d['value']), round(d['ms_per_step'],2), d['clocks']['sm_mhz'], round(d['roofline']['ms_per_launch'],3), round(d['roofline']['alone']['ms_per_launch'],3))"
done
