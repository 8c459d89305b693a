set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r1
nvidia-smi -L > gpurun_out/r1/gpus.txt
git_sha=$(cat tools/gpu/sha.txt)
(echo "# pytest -m gpu on 4x B200 at $git_sha"; timeout 1500 python -m pytest tests -m gpu -q -rs 2>&1; echo rc=$?) > gpurun_out/r1/pytest_gpu4.log 2>&1
timeout 300 python bench.py > gpurun_out/r1/bench_c3_n1.json 2> gpurun_out/r1/bench_c3_n1.err
timeout 300 python bench.py --config c1 --no-cpu > gpurun_out/r1/bench_c1.json 2> gpurun_out/r1/bench_c1.err
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 4 --steps 20 --warmup 5 --no-e2e > gpurun_out/r1/bench_c3_n4.json 2> gpurun_out/r1/bench_c3_n4.err
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 4 --steps 20 --warmup 5 --no-e2e --transport nccl > gpurun_out/r1/bench_c3_n4_nccl.json 2> gpurun_out/r1/bench_c3_n4_nccl.err
