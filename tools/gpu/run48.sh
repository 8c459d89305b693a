# 4-GPU call at the final HEAD: full pytest -m gpu, then the default bench at N=4 and N=1
cd $GRAFT_REPO_ROOT
O=gpurun_out/r48; mkdir -p $O
sha=$(cat tools/gpu/sha.txt)
(echo "# pytest -m gpu on 4x B200 at $sha"; timeout 1500 python -m pytest tests -m gpu -q -rs 2>&1; echo rc=$?) > $O/pytest_gpu4.log 2>&1
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 30411 bench.py --gpus 4 --steps 20 --warmup 5 > $O/bench_c3_n4.json 2> $O/bench_c3_n4.err
timeout 400 python bench.py > $O/bench_c3_n1.json 2> $O/bench_c3_n1.err
