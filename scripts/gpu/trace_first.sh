# role timelines of the rate-coded first layers (C3 / C2 layer 0) + an ncu capture of C3 L0
bash scripts/gpu/trace.sh "C3 0 tac 8 1024" "C2 0 tac 4 256" "C3 0 dense 1 1024" "C5 0 tactp 4 256"
python -m paper_2603_13810_b200.build > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_conv_lif -s 1 -c 1 -o gpurun_out/c3l0_r02 -f python scripts/profile_layer.py --config C3 --layer 0 --mode tac --K 8 --B 1024 --iters 2 --no-counts > gpurun_out/ncu_c3l0.log 2>&1; echo "ncu_rc=$?"
