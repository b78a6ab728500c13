# ncu --set full with source counters: C5 layer 0 (B=1024) and C3 layer 0 (TAC K=8, B=1024)
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_conv_lif -s 1 -c 1 -o gpurun_out/c5l0 -f python scripts/profile_layer.py --config C5 --layer 0 --B 1024 --iters 2 --no-counts > gpurun_out/ncu_c5l0.log 2>&1; echo "ncu_rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_conv_lif -s 1 -c 1 -o gpurun_out/c3l0 -f python scripts/profile_layer.py --config C3 --layer 0 --mode tac --K 8 --B 1024 --iters 2 --no-counts > gpurun_out/ncu_c3l0.log 2>&1; echo "ncu_rc=$?"
