# 1-GPU call: atomics-based block_finish + per-role LOCAL tickets: parity, C1/C2/C3 lines, C2 waves
cd $GRAFT_REPO_ROOT
O=gpurun_out/r5; mkdir -p $O
(timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_rounds.py tests/test_gpu_acceptance.py -m gpu -q -x 2>&1; echo rc=$?) > $O/pytest_1gpu.log 2>&1
timeout 300 python bench.py --config c1 --no-cpu > $O/bench_c1.json 2> $O/bench_c1.err
timeout 300 python bench.py --config c2 --no-cpu --no-e2e > $O/bench_c2.json 2> $O/bench_c2.err
timeout 300 python bench.py --no-cpu --no-e2e > $O/bench_c3.json 2> $O/bench_c3.err
timeout 400 python tools/tune_fused.py --mode 1 --n 125000000 --variants 0,4,5 --waves 4,8,32 --reps 3 --iters 60 > $O/tune_c2_f32.jsonl 2> $O/tune_c2_f32.err
for mi in 8 32; do CO2_MIN_CTA_ITERS=$mi timeout 300 python bench.py --config c2 --no-cpu --no-e2e > $O/bench_c2_mi$mi.json 2> $O/bench_c2_mi$mi.err; done
