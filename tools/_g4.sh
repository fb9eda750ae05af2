mkdir -p gpurun_out/s7
timeout 900 python -m pytest tests -m gpu -q -s > gpurun_out/s7/pytest_gpu.txt 2>&1
bash tools/_bench_ab.sh C4 base int8lo2 > gpurun_out/s7/ab_c4.txt 2>&1
bash tools/_bench_ab.sh C3 base int8lo2 > gpurun_out/s7/ab_c3.txt 2>&1
