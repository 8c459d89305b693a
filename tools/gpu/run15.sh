# 1-GPU call: LOCAL round with static first tiles -- round tests, C1 bench
cd $GRAFT_REPO_ROOT
O=gpurun_out/r15; mkdir -p $O
(timeout 900 python -m pytest tests/test_gpu_rounds.py tests/test_gpu_acceptance.py -m gpu -q -x 2>&1; echo rc=$?) > $O/pytest.log 2>&1
for r in 1 2; do timeout 300 python bench.py --config c1 --no-cpu --steps 40 > $O/bench_c1_r$r.json 2> $O/bench_c1_r$r.err; done
for tv in 2 8; do CO2_LOCAL_ROUND_TV=$tv timeout 300 python bench.py --config c1 --no-cpu --steps 40 > $O/bench_c1_tv$tv.json 2> $O/bench_c1_tv$tv.err; done
