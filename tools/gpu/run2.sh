# 2-GPU call: bulk-copy step parity + tuning, baseline kernels, N=2 split schedule per variant,
# C5 sweep at N=2 (both transports).
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2; mkdir -p $O
(timeout 900 python -m pytest tests -m gpu -q -x -k "bulk or baseline" 2>&1; echo rc=$?) > $O/pytest_bulk.log 2>&1
timeout 600 python tools/tune_fused.py --mode 2 --n 1300000000 --variants 0,10,11,12,13,14 --reps 3 > $O/tune_c3_bf16.jsonl 2>$O/tune_c3_bf16.err
timeout 300 python tools/tune_fused.py --mode 1 --n 125000000 --variants 0,10,11,12,13,14 --reps 5 --iters 60 > $O/tune_c2_f32.jsonl 2>$O/tune_c2_f32.err
timeout 600 python tools/tune_fused.py --mode 0 --n 650000000 --variants 0,4,10,11,12 --reps 3 > $O/tune_f64.jsonl 2>$O/tune_f64.err
timeout 300 python tools/baseline_bench.py > $O/baseline_bench.jsonl 2>$O/baseline_bench.err
for rep in 1 2; do
for v in 0 10 12 13; do
CO2_FUSED_VARIANT=$v timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $((29600+v+rep*20)) bench.py --gpus 2 --steps 20 --warmup 5 --no-e2e > $O/bench_c3_n2_v${v}_r$rep.json 2> $O/bench_c3_n2_v${v}_r$rep.err
done; done
for v in 0 10; do
CO2_FUSED_VARIANT=$v timeout 300 python bench.py --config c2 --no-e2e --no-cpu --steps 50 > $O/bench_c2_n1_v$v.json 2> $O/bench_c2_n1_v$v.err
done
for t in p2p nccl; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29540 tools/overlap_sweep.py --transport $t --out $O/overlap_$t.jsonl > $O/overlap_$t.log 2>&1
done
