# 4-GPU call: grid-independent P2P exit barrier + adaptive reduce occupancy -- multi-GPU tests, C3 N=4 bench, C5 GEMM sweep adaptive
cd $GRAFT_REPO_ROOT
O=gpurun_out/r42; mkdir -p $O
(timeout 1500 python -m pytest tests/test_gpu_multi.py -m gpu -q -x 2>&1; echo rc=$?) > $O/pytest_multi.log 2>&1
P=30100
for ad in 0 1; do P=$((P+1)); CO2_P2P_ADAPT=$ad timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $P bench.py --gpus 4 --steps 20 --warmup 5 --no-e2e --no-cpu > $O/bench_c3_n4_adapt$ad.json 2> $O/bench_c3_n4_adapt$ad.err; done
P=$((P+1)); CO2_P2P_ADAPT=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $P tools/overlap_sweep.py --transport p2p --inner gemm --out $O/overlap_p2p_n4_gemm_adapt.jsonl > $O/overlap_p2p_n4_gemm_adapt.log 2>&1
