# round-2 evidence: full GPU suite, sweep, bench line, ncu launch list of the bench, ncu --set full of C5 L0 / L1 and C3 L0
bash scripts/gpu/tests.sh
timeout 1500 python scripts/sweep.py --out gpurun_out/sweep_r02.jsonl > gpurun_out/sweep.log 2>&1; echo "sweep_rc=$?"; tail -2 gpurun_out/sweep.log
timeout 600 python bench.py > gpurun_out/bench_r02.json 2> gpurun_out/bench.err; echo "bench_rc=$?"; tail -c 400 gpurun_out/bench_r02.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'tc_conv|tc_zero|pack_kernel|simt|fc_lif' --csv --log-file gpurun_out/launches_r02.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo "ncu_launch_rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_conv_lif -s 1 -c 1 -o gpurun_out/c5l0_full_r02 -f python scripts/profile_layer.py --config C5 --layer 0 --B 2048 --iters 2 --no-counts > gpurun_out/ncu1.log 2>&1; echo "ncu_l0_rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_conv_lif -s 1 -c 1 -o gpurun_out/c5l1_full_r02 -f python scripts/profile_layer.py --config C5 --layer 1 --B 2048 --iters 2 --no-counts > gpurun_out/ncu2.log 2>&1; echo "ncu_l1_rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_conv_lif -s 1 -c 1 -o gpurun_out/c3l0_full_r02 -f python scripts/profile_layer.py --config C3 --layer 0 --mode tac --K 8 --B 1024 --iters 2 --no-counts > gpurun_out/ncu3.log 2>&1; echo "ncu_c3_rc=$?"
