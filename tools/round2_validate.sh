# One GPU call for the round-2 evidence: the full -m gpu suite (log kept), smoke(), bench lines for
# C4 (+ the reference arm) / C2 / C3, and the round profile (ncu launch lists + full captures).
out=${1:-gpurun_out/r2v}; mkdir -p $out
timeout 1500 python -m pytest tests -m gpu -q -s -p no:randomly > $out/gputest.log 2>&1; tail -3 $out/gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; tail -1 $out/smoke.log
timeout 600 python bench.py --impl reference --steps 5 --warmup 1 > $out/bench_C4_reference.json 2> $out/bench_ref.err
bash tools/round_profile.sh $out > /dev/null 2>&1
for c in C4 C2 C3; do python -c "import json;d=json.load(open('$out/bench_$c.json'));print('$c', round(d['value']), round(d['ms_per_step'],2), d['clocks']['sm_mhz'], round(d['roofline']['frac'],3), round(d['e2e']['value']))"; done
python -c "import json;d=json.load(open('$out/bench_C4_reference.json'));print('ref', d['value'], d['cpu_baseline']['sample'][:120])"
