# 1-GPU call at HEAD (final kernels): driver-like default bench, ncu launch list, ncu --set full of the C3 / C2 / C1 kernels
cd $GRAFT_REPO_ROOT
O=gpurun_out/r37; mkdir -p $O
timeout 400 python bench.py --steps 20 --warmup 5 > $O/bench_c3_default.json 2> $O/bench_c3_default.err
timeout 400 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_c3.csv python bench.py --steps 2 --warmup 1 > $O/launches_c3.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused_step_kernel -s 3 -c 1 -o /tmp/c3_fused_step python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > $O/c3_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused_step_kernel -s 3 -c 1 -o /tmp/c2_fused_step python bench.py --config c2 --steps 2 --warmup 3 --no-e2e --no-cpu > $O/c2_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:local_round_kernel -s 8 -c 1 -o /tmp/c1_local_round python bench.py --config c1 --no-cpu --steps 4 --warmup 3 > $O/c1_full.log 2>&1
for k in c3_fused_step c2_fused_step c1_local_round; do ncu -i /tmp/$k.ncu-rep --page raw --csv > $O/${k}_raw.csv 2>/dev/null; ncu -i /tmp/$k.ncu-rep --page details > $O/${k}_details.txt 2>/dev/null; ncu -i /tmp/$k.ncu-rep --page source --csv --print-source sass > $O/${k}_source.csv 2>/dev/null; done
