# ncu --set full with source counters on C5 layer 0 (the bench's dominant kernel)
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_conv_lif -s 1 -c 1 -o gpurun_out/c5l0 -f python scripts/profile_layer.py --config C5 --layer 0 --B ${1:-2048} --iters 2 --no-counts > gpurun_out/ncu_c5l0.log 2>&1; echo "ncu_rc=$?"
tail -3 gpurun_out/ncu_c5l0.log
