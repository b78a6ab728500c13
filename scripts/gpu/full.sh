# full GPU suite, sweep (all configs + whole networks, clocks + roofline), default bench line
bash scripts/gpu/tests.sh
timeout 1200 python scripts/sweep.py --out gpurun_out/sweep.jsonl > gpurun_out/sweep.log 2>&1; echo "sweep_rc=$?"; tail -3 gpurun_out/sweep.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench_rc=$?"; tail -c 600 gpurun_out/bench.json; tail -3 gpurun_out/bench.err
