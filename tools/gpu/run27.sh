# 4-GPU call at HEAD: full pytest -m gpu; driver-like bench lines at N=1/2/4 (e2e on); reference arm; C1
cd $GRAFT_REPO_ROOT
O=gpurun_out/r27; mkdir -p $O
sha=$(cat tools/gpu/sha.txt)
(echo "# pytest -m gpu on 4x B200 at $sha"; timeout 1800 python -m pytest tests -m gpu -q -rs 2>&1; echo rc=$?) > $O/pytest_gpu4.log 2>&1
timeout 400 python bench.py > $O/bench_c3_n1.json 2> $O/bench_c3_n1.err
timeout 400 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err
P=29900
for w in 2 4; do P=$((P+1)); timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $w --master-addr 127.0.0.1 --master-port $P bench.py --gpus $w --steps 20 --warmup 5 > $O/bench_c3_n$w.json 2> $O/bench_c3_n$w.err; done
timeout 300 python bench.py --config c1 --no-cpu --steps 40 > $O/bench_c1.json 2> $O/bench_c1.err
timeout 300 python bench.py --config c2 --no-cpu --steps 20 > $O/bench_c2_n1.json 2> $O/bench_c2_n1.err
