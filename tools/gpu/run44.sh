# 4-GPU call: C3 N=4 x3 and N=2 with per-rank elapsed / host enqueue diagnostics
cd $GRAFT_REPO_ROOT
O=gpurun_out/r44; mkdir -p $O
P=30200
for r in 1 2 3; do P=$((P+1)); timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $P bench.py --gpus 4 --steps 20 --warmup 5 --no-e2e --no-cpu > $O/bench_c3_n4_r$r.json 2> $O/bench_c3_n4_r$r.err; done
P=$((P+1)); timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $P bench.py --gpus 2 --steps 20 --warmup 5 --no-e2e --no-cpu > $O/bench_c3_n2.json 2> $O/bench_c3_n2.err
