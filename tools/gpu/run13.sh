# 1-GPU call: kernel-timed LOCAL round (no timing events), TV sweep
cd $GRAFT_REPO_ROOT
O=gpurun_out/r13; mkdir -p $O
(timeout 900 python -m pytest tests/test_gpu_rounds.py tests/test_gpu_acceptance.py tests/test_gpu_parity.py -m gpu -q -x 2>&1; echo rc=$?) > $O/pytest.log 2>&1
for r in 1 2; do for tv in 2 4 8; do CO2_LOCAL_ROUND_TV=$tv timeout 300 python bench.py --config c1 --no-cpu > $O/bench_c1_tv${tv}_r$r.json 2> $O/bench_c1_tv${tv}_r$r.err; done; done
timeout 300 python tools/c1_gap.py > $O/c1_gap.jsonl 2> $O/c1_gap.err
