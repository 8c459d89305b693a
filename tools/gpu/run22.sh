# 4-GPU call: register-capped step (variants 6/7, <= 56 regs) + 128-thread reduce CTAs that fit beside 4 step CTAs/SM
cd $GRAFT_REPO_ROOT
O=gpurun_out/r22; mkdir -p $O
(timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "variant or fused" 2>&1; echo rc=$?) > $O/pytest.log 2>&1
for v in 0 6 7; do CO2_FUSED_VARIANT=$v timeout 300 python bench.py --no-cpu --no-e2e --steps 20 > $O/c3_n1_v$v.json 2>/dev/null; done
P=29700
for rep in 1 2; do for w in 2 4; do
for cfg in "0 256 96" "6 128 148" "6 128 96" "7 128 148" "6 256 96"; do set -- $cfg; P=$((P+1))
CO2_FUSED_VARIANT=$1 CO2_P2P_THREADS=$2 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $w --master-addr 127.0.0.1 --master-port $P bench.py --gpus $w --steps 20 --warmup 5 --no-e2e --no-cpu --max-ctas $3 > $O/c3_n${w}_v$1_t$2_c$3_r$rep.json 2>/dev/null
done; done; done
