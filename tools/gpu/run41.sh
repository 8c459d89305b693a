# 1-GPU call: bulk-copy LOCAL round (runtime stages) -- round tests, C1 A/B, ncu of the bulk kernel
cd $GRAFT_REPO_ROOT
O=gpurun_out/r41; mkdir -p $O
(CO2_LOCAL_ROUND_BULK=1 timeout 900 python -m pytest tests/test_gpu_rounds.py tests/test_gpu_acceptance.py -m gpu -q -x 2>&1; echo rc=$?) > $O/pytest_bulk1.log 2>&1
for r in 1 2; do for b in 0 1 2 3; do CO2_LOCAL_ROUND_BULK=$b timeout 300 python bench.py --config c1 --no-cpu --steps 40 > $O/c1_bulk${b}_r$r.json 2> $O/c1_bulk${b}_r$r.err; done; done
CO2_LOCAL_ROUND_BULK=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:local_round_bulk_kernel -s 8 -c 1 -o /tmp/c1_bulk python bench.py --config c1 --no-cpu --steps 4 --warmup 3 > $O/c1_bulk_ncu.log 2>&1
ncu -i /tmp/c1_bulk.ncu-rep --page details > $O/c1_bulk_details.txt 2>/dev/null; ncu -i /tmp/c1_bulk.ncu-rep --page raw --csv > $O/c1_bulk_raw.csv 2>/dev/null
