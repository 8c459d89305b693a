# 1-GPU call at the final HEAD: pytest -m gpu (single-GPU suites), driver-like default bench, C1 / C2 lines, smoke()
cd $GRAFT_REPO_ROOT
O=gpurun_out/r46; mkdir -p $O
sha=$(cat tools/gpu/sha.txt)
(echo "# pytest -m gpu on 1x B200 at $sha"; timeout 1500 python -m pytest tests -m gpu -q -rs 2>&1 | tail -15; echo rc=$?) > $O/pytest_gpu1.log 2>&1
(timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1; echo rc=$?) > $O/smoke.log 2>&1
timeout 400 python bench.py > $O/bench_c3_n1.json 2> $O/bench_c3_n1.err
timeout 300 python bench.py --config c1 --no-cpu --steps 40 > $O/bench_c1.json 2> $O/bench_c1.err
timeout 300 python bench.py --config c2 --no-cpu --steps 20 > $O/bench_c2.json 2> $O/bench_c2.err
