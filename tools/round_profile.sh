# One GPU call: bench lines for C2/C3/C4, ncu launch lists (time + DRAM bytes) of one C4 and one C2
# step, and ncu --set full captures of the attention, QKV+RoPE and gate/up+SwiGLU kernels at C4.
#   bash tools/round_profile.sh OUTDIR
out=${1:-gpurun_out/prof}; mkdir -p $out
for c in C4 C2 C3; do timeout 600 python bench.py --config $c > $out/bench_$c.json 2> $out/bench_$c.err; done
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum"
K='regex:gemm|attn|embed|head|gather|rope'
for c in C4 C2; do
  timeout 600 ncu --metrics $M --clock-control none -k "$K" -s 146 -c 146 --csv --log-file $out/launches_$c.csv \
    python tools/profile_step.py --config $c > /dev/null 2>&1
  python tools/launch_breakdown.py $out/launches_$c.csv > $out/launch_breakdown_$c.txt 2>&1
done
for k in "attn_prefix:attn" "gemm_bf16_kernel<.int.1,:qkv_rope" "gemm_bf16_kernel<.int.2,:gateup_swiglu" "gemm_bf16_kernel<.int.4,:resid_norm"; do
  pat=${k%%:*}; name=${k##*:}
  timeout 600 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k "regex:$pat" -s 30 -c 1 -o $out/${name}_c4 \
    python tools/profile_step.py --config C4 > /dev/null 2>&1
done
ls -la $out
