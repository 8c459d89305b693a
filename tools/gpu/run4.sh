# 2-GPU call: TMA bulk-copy P2P all-reduce -- parity, alone (aar_bench), and co-running with the C3 step.
cd $GRAFT_REPO_ROOT
O=gpurun_out/r4; mkdir -p $O
(timeout 900 python -m pytest tests/test_gpu_multi.py -m gpu -q -x -k "p2pbulk" 2>&1; echo rc=$?) > $O/pytest_p2pbulk.log 2>&1
for b in 0 2 4; do
CO2_P2P_BULK=$b timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $((29650+b)) tools/aar_bench.py --ctas 16,32,64,96,148 > $O/aar_n2_bulk$b.jsonl 2> $O/aar_n2_bulk$b.err
done
for rep in 1 2; do
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $((29660+rep)) bench.py --gpus 2 --steps 20 --warmup 5 --no-e2e --no-cpu > $O/bench_c3_n2_reg_r$rep.json 2> $O/bench_c3_n2_reg_r$rep.err
for b in 2 4; do for c in 32 64 148; do
CO2_P2P_BULK=$b timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $((29670+b*3+rep)) bench.py --gpus 2 --steps 20 --warmup 5 --no-e2e --no-cpu --max-ctas $c > $O/bench_c3_n2_bulk${b}_c${c}_r$rep.json 2> $O/bench_c3_n2_bulk${b}_c${c}_r$rep.err
done; done; done
timeout 400 python tools/tune_fused.py --mode 1 --n 125000000 --variants 0,3,4,5 --waves 4,8,32 --reps 3 --iters 60 > $O/tune_c2_f32.jsonl 2> $O/tune_c2_f32.err
timeout 600 python tools/tune_fused.py --mode 0 --n 1300000000 --variants 0,5 --reps 3 --iters 20 > $O/tune_c3_f64.jsonl 2> $O/tune_c3_f64.err
