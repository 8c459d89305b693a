# 4-GPU call at HEAD: full pytest -m gpu, C3/C2/C4 at N=1/2/4 (defaults), C3 N=4 CTA sweep, NCCL, C5 sweeps at N=4
cd $GRAFT_REPO_ROOT
O=gpurun_out/r18; mkdir -p $O
sha=$(cat tools/gpu/sha.txt)
nvidia-smi -L > $O/gpus.txt
(echo "# pytest -m gpu on 4x B200 at $sha"; timeout 1800 python -m pytest tests -m gpu -q -rs 2>&1; echo rc=$?) > $O/pytest_gpu4.log 2>&1
timeout 400 python bench.py > $O/bench_c3_n1.json 2> $O/bench_c3_n1.err
P=29600
run() { P=$((P+1)); timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 --master-port $P bench.py --gpus $1 --steps 20 --warmup 5 "${@:3}" > $O/$2.json 2> $O/$2.err; }
run 2 bench_c3_n2
run 4 bench_c3_n4
run 4 bench_c3_n4_nccl --transport nccl --no-e2e
for c in 128 148; do run 4 bench_c3_n4_c$c --max-ctas $c --no-e2e; done
run 2 bench_c2_n2 --config c2 --no-e2e
run 4 bench_c2_n4 --config c2 --no-e2e
run 2 bench_c4_n2 --config c4 --no-e2e
run 4 bench_c4_n4 --config c4 --no-e2e
for t in p2p nccl; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29591 tools/overlap_sweep.py --transport $t --out $O/overlap_${t}_n4.jsonl > $O/overlap_${t}_n4.log 2>&1
done
