# 4-GPU call: C5 tau sweeps with the tensor-core GEMM inner step (N=2, N=4; P2P, NCCL) and the HBM one at N=2
cd $GRAFT_REPO_ROOT
O=gpurun_out/r35; mkdir -p $O
P=29960
for w in 4 2; do for t in p2p nccl; do P=$((P+1))
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $w --master-addr 127.0.0.1 --master-port $P tools/overlap_sweep.py --transport $t --inner gemm --out $O/overlap_${t}_n${w}_gemm.jsonl > $O/overlap_${t}_n${w}_gemm.log 2>&1
done; done
for t in p2p nccl; do P=$((P+1))
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $P tools/overlap_sweep.py --transport $t --out $O/overlap_${t}_n2_hbm.jsonl > $O/overlap_${t}_n2_hbm.log 2>&1
done
