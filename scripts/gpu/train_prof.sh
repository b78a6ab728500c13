python -m paper_2603_13810_b200.build > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/train_launches.csv python bench.py --train --steps 1 --warmup 0 --config C4 --mode tactp --K 2 --B 16 > gpurun_out/train_ncu.log 2>&1; echo "rc=$?"
