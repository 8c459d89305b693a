# 4-GPU call at the final HEAD: full pytest -m gpu; driver-like lines N=1/2/4; c3f64, c2, c1, c4; reference arm
cd $GRAFT_REPO_ROOT
O=gpurun_out/r43; mkdir -p $O
sha=$(cat tools/gpu/sha.txt)
(echo "# pytest -m gpu on 4x B200 at $sha"; timeout 1800 python -m pytest tests -m gpu -q -rs 2>&1; echo rc=$?) > $O/pytest_gpu4.log 2>&1
timeout 400 python bench.py > $O/bench_c3_n1.json 2> $O/bench_c3_n1.err
P=29990
for w in 2 4; do P=$((P+1)); timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $w --master-addr 127.0.0.1 --master-port $P bench.py --gpus $w --steps 20 --warmup 5 > $O/bench_c3_n$w.json 2> $O/bench_c3_n$w.err; done
timeout 600 python bench.py --config c3f64 --no-cpu --no-e2e --steps 10 > $O/bench_c3f64.json 2> $O/bench_c3f64.err
timeout 300 python bench.py --config c2 --no-cpu --steps 20 > $O/bench_c2_n1.json 2> $O/bench_c2_n1.err
timeout 300 python bench.py --config c1 --no-cpu --steps 40 > $O/bench_c1.json 2> $O/bench_c1.err
for w in 2 4; do P=$((P+1)); timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $w --master-addr 127.0.0.1 --master-port $P bench.py --gpus $w --config c4 --steps 10 --warmup 3 --no-e2e --no-cpu > $O/bench_c4_n$w.json 2> $O/bench_c4_n$w.err; done
timeout 400 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err
