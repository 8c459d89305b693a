# 1-GPU call: dynamic-tile LOCAL round kernel -- round tests, C1 bench x2, c1_gap, ncu of the round kernel
cd $GRAFT_REPO_ROOT
O=gpurun_out/r10; mkdir -p $O
(timeout 900 python -m pytest tests/test_gpu_rounds.py tests/test_gpu_acceptance.py -m gpu -q -x 2>&1; echo rc=$?) > $O/pytest_rounds.log 2>&1
for r in 1 2; do timeout 300 python bench.py --config c1 --no-cpu > $O/bench_c1_r$r.json 2> $O/bench_c1_r$r.err; done
timeout 300 python tools/c1_gap.py > $O/c1_gap.jsonl 2> $O/c1_gap.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:local_round_kernel -s 4 -c 1 -o $O/c1_local_round python bench.py --config c1 --no-cpu --steps 3 --warmup 3 > $O/c1_full.log 2>&1
