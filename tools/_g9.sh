out=gpurun_out/s13; mkdir -p $out
bash tools/sanitize.sh > $out/sanitize.txt 2>&1
cp gpurun_out/sanitize_*.log $out/ 2>/dev/null
timeout 900 python bench.py --config C5 > $out/bench_C5.json 2> $out/bench_C5.err
bash tools/_bench_ab.sh C2 cur pref > $out/ab_c2.txt 2>&1
