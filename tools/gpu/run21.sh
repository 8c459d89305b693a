# 1-GPU call: A/B of the warp-uniform division fast path (ab_old = HEAD without it), interleaved
cd $GRAFT_REPO_ROOT
O=$GRAFT_REPO_ROOT/gpurun_out/r21; mkdir -p $O
for rep in 1 2; do for v in old new; do
  if [ $v = old ]; then D=ab_old; else D=.; fi
  (cd $D && timeout 300 python bench.py --config c2 --no-cpu --no-e2e > $O/c2_${v}_$rep.json 2>/dev/null)
  (cd $D && timeout 300 python bench.py --config c1 --no-cpu --steps 40 > $O/c1_${v}_$rep.json 2>/dev/null)
  (cd $D && timeout 300 python bench.py --no-cpu --no-e2e --steps 20 > $O/c3_${v}_$rep.json 2>/dev/null)
  (cd $D && timeout 300 python tools/data_regime.py --mode 1 --n 125000000 --steps 120 > $O/regime_${v}_$rep.jsonl 2>/dev/null)
done; done
