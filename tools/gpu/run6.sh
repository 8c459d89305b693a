# 4-GPU call: 64-register P2P reduce -- parity, C3 at N=2/4 over reduce CTA shapes; C1 host time
cd $GRAFT_REPO_ROOT
O=gpurun_out/r6; mkdir -p $O
(timeout 1200 python -m pytest tests/test_gpu_multi.py -m gpu -q -x 2>&1; echo rc=$?) > $O/pytest_multi.log 2>&1
timeout 300 python bench.py --config c1 --no-cpu > $O/bench_c1.json 2> $O/bench_c1.err
for w in 2 4; do for rep in 1 2; do
for cfg in "256 0" "128 148" "128 96" "256 64" "256 96"; do set -- $cfg
CO2_P2P_THREADS=$1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $w --master-addr 127.0.0.1 --master-port $((29700+w*10+rep)) bench.py --gpus $w --steps 20 --warmup 5 --no-e2e --no-cpu --max-ctas $2 > $O/bench_c3_n${w}_t$1_c$2_r$rep.json 2> $O/bench_c3_n${w}_t$1_c$2_r$rep.err
done; done; done
