python -m paper_2603_13810_b200.build > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_backward.py -x -q > gpurun_out/pytest_bwd.log 2>&1; echo "pytest_rc=$?"; tail -3 gpurun_out/pytest_bwd.log
for args in "--config C4 --mode tactp --K 2 --B 16" "--config C4 --mode tac --K 2 --B 16" "--config C3 --mode tac --K 8" "--config C3 --mode tac --K 8 --whole-net" "--config C2 --mode tac --K 4 --whole-net"; do
  timeout 600 python bench.py --train --steps 5 --warmup 2 $args 2>&1 | tail -1 >> gpurun_out/train_bench_r02.jsonl
  tail -1 gpurun_out/train_bench_r02.jsonl | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$args', round(d['ms_per_step'],3), round(d.get('speedup_vs_dense') or 0,2))"
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/train_launches.csv python bench.py --train --steps 1 --warmup 0 --config C4 --mode tactp --K 2 --B 16 > gpurun_out/train_ncu.log 2>&1; echo "ncu_rc=$?"
