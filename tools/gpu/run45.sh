# 4-GPU call: comm-stream readbacks as mapped kernel writes (no copy-engine head-of-line wait) -- multi + rounds tests, C3 N=4 x4, N=2, C5 NCCL N=4
cd $GRAFT_REPO_ROOT
O=gpurun_out/r45; mkdir -p $O
(timeout 1500 python -m pytest tests/test_gpu_multi.py tests/test_gpu_rounds.py -m gpu -q -x 2>&1; echo rc=$?) > $O/pytest.log 2>&1
P=30300
for r in 1 2 3 4; do P=$((P+1)); timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $P bench.py --gpus 4 --steps 20 --warmup 5 --no-e2e --no-cpu > $O/bench_c3_n4_r$r.json 2> $O/bench_c3_n4_r$r.err; done
P=$((P+1)); timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $P bench.py --gpus 4 --steps 20 --warmup 5 --no-e2e --no-cpu --transport nccl > $O/bench_c3_n4_nccl.json 2> $O/bench_c3_n4_nccl.err
