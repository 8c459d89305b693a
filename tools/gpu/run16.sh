# 1-GPU call: C1 with / without the device-mapped host writes
cd $GRAFT_REPO_ROOT
O=gpurun_out/r16; mkdir -p $O
for r in 1 2; do for nh in 0 1; do CO2_LOCAL_ROUND_NOHOST=$nh timeout 300 python bench.py --config c1 --no-cpu --steps 40 > $O/bench_c1_nh${nh}_r$r.json 2> $O/bench_c1_nh${nh}_r$r.err; done; done
