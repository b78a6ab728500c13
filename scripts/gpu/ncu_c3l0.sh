python -m paper_2603_13810_b200.build > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_conv_lif -s 1 -c 1 -o gpurun_out/c3l0 -f python scripts/profile_layer.py --config C3 --layer 0 --mode tac --K 8 --B 1024 --iters 2 > gpurun_out/ncu_c3l0.log 2>&1; echo "ncu_rc=$?"
tail -3 gpurun_out/ncu_c3l0.log
