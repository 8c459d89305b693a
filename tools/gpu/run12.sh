# 1-GPU call: LOCAL round with CTA claims + L2 bulk prefetch of the tile after next (U, PF variants)
cd $GRAFT_REPO_ROOT
O=gpurun_out/r12; mkdir -p $O
(timeout 900 python -m pytest tests/test_gpu_rounds.py tests/test_gpu_acceptance.py -m gpu -q -x 2>&1; echo rc=$?) > $O/pytest_rounds.log 2>&1
(CO2_LOCAL_ROUND_U=1 timeout 900 python -m pytest tests/test_gpu_rounds.py -m gpu -q -x 2>&1; echo rc=$?) > $O/pytest_rounds_u1.log 2>&1
for r in 1 2; do for u in 1 2; do for pf in 0 1; do CO2_LOCAL_ROUND_PF=$pf CO2_LOCAL_ROUND_U=$u timeout 300 python bench.py --config c1 --no-cpu > $O/bench_c1_u${u}_pf${pf}_r$r.json 2> $O/bench_c1_u${u}_pf${pf}_r$r.err; done; done; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:local_round_kernel -s 4 -c 1 -o $O/c1_local_round python bench.py --config c1 --no-cpu --steps 3 --warmup 3 > $O/c1_full.log 2>&1
