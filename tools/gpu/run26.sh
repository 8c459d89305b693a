# 2-GPU call: co2_round_host -- parity test, round-level e2e at N=1 / N=2
cd $GRAFT_REPO_ROOT
O=gpurun_out/r26; mkdir -p $O
(timeout 900 python -m pytest tests/test_gpu_rounds.py -m gpu -q -x -k "round_host or single_launch" 2>&1; echo rc=$?) > $O/pytest.log 2>&1
timeout 400 python bench.py --no-cpu --steps 20 > $O/bench_c3_n1.json 2> $O/bench_c3_n1.err
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29811 bench.py --gpus 2 --steps 20 --warmup 5 > $O/bench_c3_n2.json 2> $O/bench_c3_n2.err
timeout 400 python bench.py --config c2 --no-cpu --steps 20 > $O/bench_c2_n1.json 2> $O/bench_c2_n1.err
