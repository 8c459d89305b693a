# 1-GPU call: div_rn (zero-dividend fast path) -- parity, data regime f32/f64, C2 bench; C1 event costs
cd $GRAFT_REPO_ROOT
O=gpurun_out/r9; mkdir -p $O
timeout 300 python tools/data_regime.py --mode 1 --n 125000000 --steps 200 > $O/regime_f32.jsonl 2> $O/regime_f32.err
timeout 300 python tools/data_regime.py --mode 0 --n 62500000 --steps 200 > $O/regime_f64.jsonl 2> $O/regime_f64.err
timeout 300 python tools/c1_gap.py > $O/c1_gap.jsonl 2> $O/c1_gap.err
timeout 300 python bench.py --config c2 --no-cpu --no-e2e > $O/bench_c2.json 2> $O/bench_c2.err
(timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_rounds.py tests/test_gpu_acceptance.py tests/test_gpu_large.py -m gpu -q -x 2>&1; echo rc=$?) > $O/pytest_1gpu.log 2>&1
