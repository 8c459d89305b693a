# 4-GPU call: sharded P2P round with a copy-engine all-gather (CO2_SHARD_AG=ce) vs the fused stores
cd $GRAFT_REPO_ROOT
O=gpurun_out/r29; mkdir -p $O
(CO2_SHARD_AG=ce timeout 1200 python -m pytest tests/test_gpu_multi.py -m gpu -q -x -k "shard" 2>&1; echo rc=$?) > $O/pytest_shard_ce.log 2>&1
P=29950
for rep in 1 2; do for w in 2 4; do for ag in fused ce; do P=$((P+1))
CO2_SHARD_AG=$ag timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $w --master-addr 127.0.0.1 --master-port $P bench.py --gpus $w --config c4 --steps 10 --warmup 3 --no-e2e --no-cpu > $O/c4_n${w}_${ag}_r$rep.json 2> $O/c4_n${w}_${ag}_r$rep.err
done; done; done
