# 4-GPU call: full pytest -m gpu, C1 bench, C5 sweeps at N=2/4 (both transports), NCCL vs P2P at N=4, F64 C3 line.
cd $GRAFT_REPO_ROOT
O=gpurun_out/r3; mkdir -p $O
git_sha=$(cat tools/gpu/sha.txt)
(echo "# pytest -m gpu on 4x B200 at $git_sha"; timeout 1500 python -m pytest tests -m gpu -q -rs 2>&1; echo rc=$?) > $O/pytest_gpu4.log 2>&1
timeout 300 python bench.py --config c1 --no-cpu > $O/bench_c1.json 2> $O/bench_c1.err
timeout 600 python bench.py --config c3f64 --no-cpu > $O/bench_c3f64.json 2> $O/bench_c3f64.err
for t in p2p nccl; do
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29531 bench.py --gpus 4 --steps 20 --warmup 5 --no-e2e --transport $t > $O/bench_c3_n4_$t.json 2> $O/bench_c3_n4_$t.err
done
for w in 2 4; do for t in p2p nccl; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $w --master-addr 127.0.0.1 --master-port 2954$w tools/overlap_sweep.py --transport $t --out $O/overlap_${t}_n$w.jsonl > $O/overlap_${t}_n$w.log 2>&1
done; done
