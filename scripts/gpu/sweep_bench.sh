python -m paper_2603_13810_b200.build > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 1500 python scripts/sweep.py --out gpurun_out/sweep.jsonl > gpurun_out/sweep.log 2>&1; echo "sweep_rc=$?"; tail -2 gpurun_out/sweep.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench_rc=$?"; tail -c 300 gpurun_out/bench.json; tail -3 gpurun_out/bench.err
