# round-2 checkpoint: GPU suite, smoke, default bench line
bash scripts/gpu/tests.sh
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke_rc=$?"; tail -3 gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench_rc=$?"; tail -c 3000 gpurun_out/bench.json; tail -5 gpurun_out/bench.err
