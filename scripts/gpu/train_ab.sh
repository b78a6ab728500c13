python -m paper_2603_13810_b200.build > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_backward.py -x -q > gpurun_out/pytest_bwd.log 2>&1; echo "pytest_rc=$?"; tail -3 gpurun_out/pytest_bwd.log
for args in "--config C4 --mode tactp --K 2 --B 16" "--config C4 --mode tac --K 2 --B 16" "--config C3 --mode tac --K 8" "--config C3 --mode tac --K 8 --whole-net"; do
  a=$(timeout 600 python bench.py --train --steps 3 --warmup 1 $args 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],3), round(d.get('speedup_vs_dense') or 0,2))")
  b=$(TACSNN_NO_DGRAD_TC=1 TACSNN_NO_WGRAD_TC=1 timeout 600 python bench.py --train --steps 3 --warmup 1 $args 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],3), round(d.get('speedup_vs_dense') or 0,2))")
  echo "$args: tc $a | simt $b"
done
