# 1-GPU call: programmatic dependent launch of the LOCAL round kernel (PDL 0/1, with / without the fin event)
cd $GRAFT_REPO_ROOT
O=gpurun_out/r24; mkdir -p $O
(timeout 900 python -m pytest tests/test_gpu_rounds.py tests/test_gpu_acceptance.py -m gpu -q -x 2>&1; echo rc=$?) > $O/pytest.log 2>&1
for r in 1 2; do for cfg in "0 0" "1 0" "1 1"; do set -- $cfg
CO2_LOCAL_ROUND_PDL=$1 CO2_LOCAL_ROUND_NOFIN=$2 timeout 300 python bench.py --config c1 --no-cpu --steps 40 > $O/c1_pdl$1_nofin$2_r$r.json 2> $O/c1_pdl$1_nofin$2_r$r.err
done; done
