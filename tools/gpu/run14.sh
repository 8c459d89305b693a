# 1-GPU call: C1 bench with rotating jobs (inputs > L2, rounds back to back); launch list
cd $GRAFT_REPO_ROOT
O=gpurun_out/r14; mkdir -p $O
for r in 1 2; do timeout 300 python bench.py --config c1 --no-cpu --steps 40 > $O/bench_c1_r$r.json 2> $O/bench_c1_r$r.err; done
for tv in 2 6; do CO2_LOCAL_ROUND_TV=$tv timeout 300 python bench.py --config c1 --no-cpu --steps 40 > $O/bench_c1_tv$tv.json 2> $O/bench_c1_tv$tv.err; done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:local_round_kernel -c 30 --csv --log-file $O/c1_launches.csv python bench.py --config c1 --no-cpu --steps 8 --warmup 3 > $O/c1_ncu.log 2>&1
