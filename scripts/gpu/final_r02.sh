# round-2 final evidence: GPU suite, smoke, sweep, bench line, training bench, ncu launch list of the bench
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/pytest_final.log 2>&1; echo "pytest_rc=$?"; tail -2 gpurun_out/pytest_final.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke_rc=$?"; tail -1 gpurun_out/smoke.log
timeout 1500 python scripts/sweep.py --out gpurun_out/sweep_r02d.jsonl > gpurun_out/sweep.log 2>&1; echo "sweep_rc=$?"
timeout 600 python bench.py > gpurun_out/bench_r02d.json 2> gpurun_out/bench.err; echo "bench_rc=$?"
for args in "--config C3 --mode tac --K 8" "--config C3 --mode tac --K 8 --whole-net" "--config C2 --mode tac --K 4 --whole-net" "--config C4 --mode tactp --K 2 --B 16" "--config C4 --mode tac --K 2 --B 16"; do
  timeout 600 python bench.py --train --steps 5 --warmup 3 $args 2>&1 | tail -1 >> gpurun_out/train_bench_r02e.jsonl
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'tc_conv|tc_zero|pack_kernel|simt|fc_lif' --csv --log-file gpurun_out/launches_r02d.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo "ncu_launch_rc=$?"
