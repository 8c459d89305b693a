# 1-GPU call: fp32 data-regime check (evolved vs fresh inputs) and the C1 event/kernel gap
cd $GRAFT_REPO_ROOT
O=gpurun_out/r8; mkdir -p $O
timeout 300 python tools/data_regime.py --mode 1 --n 125000000 --steps 300 > $O/regime_f32.jsonl 2> $O/regime_f32.err
timeout 300 python tools/data_regime.py --mode 2 --n 125000000 --steps 300 > $O/regime_bf16.jsonl 2> $O/regime_bf16.err
timeout 300 python tools/c1_gap.py > $O/c1_gap.jsonl 2> $O/c1_gap.err
