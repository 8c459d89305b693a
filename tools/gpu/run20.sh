# 1-GPU call: warp-uniform division fast path + cheaper diagnostics -- parity, C1/C2/C3 lines, regime
cd $GRAFT_REPO_ROOT
O=gpurun_out/r20; mkdir -p $O
(timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_rounds.py tests/test_gpu_acceptance.py tests/test_gpu_large.py -m gpu -q -x 2>&1; echo rc=$?) > $O/pytest.log 2>&1
for r in 1 2; do timeout 300 python bench.py --config c1 --no-cpu --steps 40 > $O/bench_c1_r$r.json 2> $O/bench_c1_r$r.err; done
timeout 300 python bench.py --config c2 --no-cpu --no-e2e > $O/bench_c2.json 2> $O/bench_c2.err
timeout 300 python bench.py --no-cpu --no-e2e > $O/bench_c3.json 2> $O/bench_c3.err
timeout 300 python tools/data_regime.py --mode 1 --n 125000000 --steps 200 > $O/regime_f32.jsonl 2> $O/regime_f32.err
