# A/B: round-1 tree (_ab/r1, built lib) vs current tree, same box, round robin
python -m paper_2603_13810_b200.build > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
for rep in 1 2; do
  for L in 0 1; do
    a=$(cd _ab/r1 && python scripts/profile_layer.py --config C5 --layer $L --B 512 --iters 5 2>&1 | grep " ms " | tail -3 | awk '{print $1}' | tr '\n' ' ')
    b=$(python scripts/profile_layer.py --config C5 --layer $L --B 512 --iters 5 2>&1 | grep " ms " | tail -3 | awk '{print $1}' | tr '\n' ' ')
    echo "rep $rep L$L r1: $a | now: $b"
  done
done
# micro-benchmarks of the LIF instruction mix
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/pipe_rates scripts/micro/pipe_rates.cu && /tmp/pipe_rates > gpurun_out/pipe_rates.txt 2>&1
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/lif_micro scripts/micro/lif_micro.cu && /tmp/lif_micro > gpurun_out/lif_micro.txt 2>&1
cat gpurun_out/pipe_rates.txt gpurun_out/lif_micro.txt
# ncu source-level capture of C5 layer 0 (current tree)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_conv_lif -s 1 -c 1 -o gpurun_out/c5l0_r02 -f python scripts/profile_layer.py --config C5 --layer 0 --B 256 --iters 2 > gpurun_out/ncu_c5l0.log 2>&1; echo "ncu_rc=$?"
