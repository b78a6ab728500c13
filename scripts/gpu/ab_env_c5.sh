# A/B of an environment toggle ($AB_ENV) on C5 layers 0 (B=512) and C4 L0, plus DVS first-layer parity
python -m paper_2603_13810_b200.build > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests -x -q -m gpu -k "layer_parity or split or real_input or config_stack or T25 or agg or runtime or prescale or exhaustive or chaining or reset" > gpurun_out/pytest_q.log 2>&1; echo "pytest_rc=$?"; tail -2 gpurun_out/pytest_q.log
for rep in 1 2; do
  for c in "C5 0 tactp 4 512" "C4 0 tactp 2 64" "C4 0 tac 2 64" "C5 0 dense 1 256"; do set -- $c
    a=$(python scripts/profile_layer.py --config $1 --layer $2 --mode $3 --K $4 --B $5 --iters 5 --no-counts 2>&1 | grep " ms " | tail -3 | awk '{print $1}' | tr '\n' ' ')
    b=$(env $AB_ENV python scripts/profile_layer.py --config $1 --layer $2 --mode $3 --K $4 --B $5 --iters 5 --no-counts 2>&1 | grep " ms " | tail -3 | awk '{print $1}' | tr '\n' ' ')
    echo "rep $rep $c: now $a | $AB_ENV $b"
  done
done
