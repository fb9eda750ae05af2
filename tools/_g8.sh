out=gpurun_out/s12; mkdir -p $out
timeout 600 python -m pytest tests/test_ops_gpu.py tests/test_parity_gpu.py -q > $out/pytest.txt 2>&1
bash tools/_bench_ab.sh C2 cur pref; bash tools/_bench_ab.sh C3 cur pref > $out/ab_c2.txt 2>&1
bash tools/_bench_ab.sh C4 cur pref > $out/ab_c4.txt 2>&1
