python -m paper_2603_13810_b200.build > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests -x -q -m gpu -k "C1 or mnist or T25 or runtime_group or exhaustive or rgb or cin6 or prescale or agg_weights or config_stack or real_input or backward" > gpurun_out/pytest_ws.log 2>&1; echo "pytest_rc=$?"; tail -3 gpurun_out/pytest_ws.log
for v in 0 1; do
  for c in "C3 0 tac 8 1024" "C2 0 tac 4 256" "C2 0 tac 8 256" "C3 0 dense 1 1024" "C3 1 tac 8 1024" "C2 1 tac 4 256" "C5 0 tactp 4 256"; do set -- $c
    t=$(TACSNN_NO_WARP_STAGE=$v python scripts/profile_layer.py --config $1 --layer $2 --mode $3 --K $4 --B $5 --iters 6 2>&1 | grep " ms " | tail -3 | awk '{print $1}' | tr '\n' ' ')
    echo "no_ws=$v $c: $t"
  done
done
