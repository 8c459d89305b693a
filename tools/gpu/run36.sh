# 4-GPU call: P2P reduce CTA count vs interference with the GEMM inner step (N=4)
cd $GRAFT_REPO_ROOT
O=gpurun_out/r36; mkdir -p $O
P=29980
for c in 24 48 96; do P=$((P+1))
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $P tools/overlap_sweep.py --transport p2p --inner gemm --max-ctas $c --taus 1,2,4,12,32 --out $O/overlap_p2p_n4_gemm_c$c.jsonl > $O/overlap_p2p_n4_gemm_c$c.log 2>&1
done
