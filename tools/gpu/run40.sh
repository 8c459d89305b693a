# 1-GPU call: bulk-copy LOCAL round kernel (CO2_LOCAL_ROUND_BULK=1|2) -- round tests, C1 bench A/B
cd $GRAFT_REPO_ROOT
O=gpurun_out/r40; mkdir -p $O
for b in 1 2; do (CO2_LOCAL_ROUND_BULK=$b timeout 900 python -m pytest tests/test_gpu_rounds.py tests/test_gpu_acceptance.py -m gpu -q -x 2>&1; echo rc=$?) > $O/pytest_bulk$b.log 2>&1; done
for r in 1 2; do for b in 0 1 2; do CO2_LOCAL_ROUND_BULK=$b timeout 300 python bench.py --config c1 --no-cpu --steps 40 > $O/c1_bulk${b}_r$r.json 2> $O/c1_bulk${b}_r$r.err; done; done
