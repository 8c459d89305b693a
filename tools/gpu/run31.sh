# 1-GPU call: A/B of div_rn_nz (known-normal divisors) + fmin/fmax diagnostics; parity
cd $GRAFT_REPO_ROOT
O=$GRAFT_REPO_ROOT/gpurun_out/r31; mkdir -p $O
(timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_rounds.py tests/test_gpu_acceptance.py tests/test_gpu_large.py -m gpu -q -x 2>&1; echo rc=$?) > $O/pytest.log 2>&1
for rep in 1 2; do for v in old new; do
  if [ $v = old ]; then D=ab_old; else D=.; fi
  (cd $D && timeout 300 python bench.py --config c1 --no-cpu --steps 40 > $O/c1_${v}_$rep.json 2>/dev/null)
  (cd $D && timeout 300 python bench.py --config c2 --no-cpu --no-e2e > $O/c2_${v}_$rep.json 2>/dev/null)
  (cd $D && timeout 300 python bench.py --no-cpu --no-e2e --steps 20 > $O/c3_${v}_$rep.json 2>/dev/null)
done; done
