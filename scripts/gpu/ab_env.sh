# A/B of an environment toggle ($AB_ENV, e.g. TACSNN_NO_PROD_REFILL=1) on the first layers
python -m paper_2603_13810_b200.build > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests -x -q -m gpu -k "mnist or C2 or C3 or C1 or T25 or agg_weights or runtime_group or prescale or exhaustive or split or real_input" > gpurun_out/pytest_q.log 2>&1; echo "pytest_rc=$?"; tail -2 gpurun_out/pytest_q.log
for rep in 1 2; do
  for c in "C3 0 tac 8 1024" "C2 0 tac 4 256" "C3 0 dense 1 1024" "C2 0 tac 8 256"; do set -- $c
    a=$(python scripts/profile_layer.py --config $1 --layer $2 --mode $3 --K $4 --B $5 --iters 6 --no-counts 2>&1 | grep " ms " | tail -3 | awk '{print $1}' | tr '\n' ' ')
    b=$(env $AB_ENV python scripts/profile_layer.py --config $1 --layer $2 --mode $3 --K $4 --B $5 --iters 6 --no-counts 2>&1 | grep " ms " | tail -3 | awk '{print $1}' | tr '\n' ' ')
    echo "rep $rep $c: now $a | $AB_ENV $b"
  done
done
