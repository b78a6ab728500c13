# round-2 final evidence (after the high-warp-id epilogue): bench line, ncu launch list, ncu --set full of C5 L0
timeout 600 python bench.py > gpurun_out/bench_r02e.json 2> gpurun_out/bench.err; echo "bench_rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'tc_conv|tc_zero|pack_kernel|simt|fc_lif' --csv --log-file gpurun_out/launches_r02e.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo "ncu_launch_rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_conv_lif -s 1 -c 1 -o gpurun_out/c5l0_full_r02e -f python scripts/profile_layer.py --config C5 --layer 0 --B 2048 --iters 2 --no-counts > gpurun_out/ncu1.log 2>&1; echo "ncu_l0_rc=$?"
