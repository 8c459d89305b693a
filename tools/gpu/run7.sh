# 1-GPU call: C2 size sweep (fixed cost vs per-byte rate against a copy), C1 kernel vs event gap, ncu of both
cd $GRAFT_REPO_ROOT
O=gpurun_out/r7; mkdir -p $O
nvidia-smi --query-gpu=clocks.sm,clocks.mem,power.draw,temperature.gpu,clocks_throttle_reasons.active --format=csv -lms 200 > $O/smi.csv 2>&1 &
SMI=$!
timeout 400 python tools/size_sweep.py --mode 1 --sizes 31250000,62500000,125000000,250000000,500000000 > $O/size_f32.jsonl 2> $O/size_f32.err
timeout 400 python tools/size_sweep.py --mode 2 --sizes 62500000,125000000,250000000,650000000 > $O/size_bf16.jsonl 2> $O/size_bf16.err
timeout 300 python bench.py --config c1 --no-cpu > $O/bench_c1.json 2> $O/bench_c1.err
timeout 300 python bench.py --config c2 --no-cpu --no-e2e > $O/bench_c2.json 2> $O/bench_c2.err
kill $SMI
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file $O/c1_launches.csv python bench.py --config c1 --no-cpu --steps 10 --warmup 3 > $O/c1_ncu.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:local_round_kernel -s 4 -c 1 -o $O/c1_local_round python bench.py --config c1 --no-cpu --steps 3 --warmup 3 > $O/c1_full.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fused_step_kernel -s 6 -c 1 -o $O/c2_fused_step python bench.py --config c2 --no-cpu --no-e2e --steps 3 --warmup 3 > $O/c2_full.log 2>&1
