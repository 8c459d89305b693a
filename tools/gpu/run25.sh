# 1-GPU call: PDL trigger at entry (2) vs after the tiles (1); TV 2/4/6
cd $GRAFT_REPO_ROOT
O=gpurun_out/r25; mkdir -p $O
for r in 1 2; do for cfg in "1 4" "2 4" "1 6" "2 6" "2 2"; do set -- $cfg
CO2_LOCAL_ROUND_PDL=$1 CO2_LOCAL_ROUND_TV=$2 timeout 300 python bench.py --config c1 --no-cpu --steps 40 > $O/c1_pdl$1_tv$2_r$r.json 2> $O/c1_pdl$1_tv$2_r$r.err
done; done
(CO2_LOCAL_ROUND_PDL=2 timeout 900 python -m pytest tests/test_gpu_rounds.py -m gpu -q -x 2>&1; echo rc=$?) > $O/pytest_pdl2.log 2>&1
