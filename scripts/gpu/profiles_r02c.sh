timeout 900 python -m pytest tests -q -m gpu > gpurun_out/pytest_final.log 2>&1; echo "pytest_rc=$?"; tail -2 gpurun_out/pytest_final.log
# round-2 (second half) evidence: sweep, bench line, training bench, ncu launch list of the bench,
# ncu --set full of C5 L0 / L1 and C3 L0 (built library travels in-tree)
timeout 1500 python scripts/sweep.py --out gpurun_out/sweep_r02c.jsonl > gpurun_out/sweep.log 2>&1; echo "sweep_rc=$?"; tail -2 gpurun_out/sweep.log
timeout 600 python bench.py > gpurun_out/bench_r02c.json 2> gpurun_out/bench.err; echo "bench_rc=$?"; tail -c 400 gpurun_out/bench_r02c.json
for args in "--config C3 --mode tac --K 8" "--config C3 --mode tac --K 8 --whole-net" "--config C2 --mode tac --K 4 --whole-net" "--config C4 --mode tactp --K 2 --B 16" "--config C4 --mode tac --K 2 --B 16"; do
  timeout 600 python bench.py --train --steps 5 --warmup 3 $args 2>&1 | tail -1 >> gpurun_out/train_bench_r02d.jsonl
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'tc_conv|tc_zero|pack_kernel|simt|fc_lif' --csv --log-file gpurun_out/launches_r02c.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo "ncu_launch_rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_conv_lif -s 1 -c 1 -o gpurun_out/c5l0_full_r02c -f python scripts/profile_layer.py --config C5 --layer 0 --B 2048 --iters 2 --no-counts > gpurun_out/ncu1.log 2>&1; echo "ncu_l0_rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_conv_lif -s 1 -c 1 -o gpurun_out/c5l1_full_r02c -f python scripts/profile_layer.py --config C5 --layer 1 --B 2048 --iters 2 --no-counts > gpurun_out/ncu2.log 2>&1; echo "ncu_l1_rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_conv_lif -s 1 -c 1 -o gpurun_out/c3l0_full_r02c -f python scripts/profile_layer.py --config C3 --layer 0 --mode tac --K 8 --B 1024 --iters 2 --no-counts > gpurun_out/ncu3.log 2>&1; echo "ncu_c3_rc=$?"
