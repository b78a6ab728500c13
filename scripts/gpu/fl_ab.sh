python -m paper_2603_13810_b200.build > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 1200 python -m pytest tests -q -m gpu -k "first_layer or C1 or mnist or T25 or exhaustive or config_stack or whole_mnist or backward or graph or real_input" > gpurun_out/pytest_fl.log 2>&1; echo "pytest_rc=$?"; tail -3 gpurun_out/pytest_fl.log
for c in "C3 0 tac 8 1024" "C2 0 tac 4 256" "C2 0 tac 8 256" "C3 0 dense 1 1024" "C1 0 tac 4 4" "C1 0 dense 1 4"; do set -- $c
  for e in simt tcgen05; do
    t=$(python scripts/profile_layer.py --config $1 --layer $2 --mode $3 --K $4 --B $5 --iters 6 --engine $e 2>&1 | grep " ms " | tail -3 | awk '{print $1}' | tr '\n' ' ')
    echo "$e $c: $t"
  done
done
