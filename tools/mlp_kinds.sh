# fused layer tail restricted to one tile kind (no dependencies), to compare with the standalone GEMMs
for k in 1 2 4 7; do PF_MLP_NODEP=1 PF_MLP_KINDS=$k python tools/mlp_probe.py C4 1,4,8 2>&1 | grep -E "rows|three" | cut -c1-70 | sed "s/^/kinds=$k /"; done
