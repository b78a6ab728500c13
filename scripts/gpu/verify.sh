# verify the in-tree build on a B200: full GPU tests, smoke, bench, training bench
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/pytest.log 2>&1; echo "pytest_rc=$?"
tail -5 gpurun_out/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke_rc=$?"; tail -2 gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench_rc=$?"; cat gpurun_out/bench.json | head -c 3000
for args in "--config C3 --mode tac --K 8" "--config C3 --mode tac --K 8 --whole-net" "--config C4 --mode tactp --K 2 --B 16" "--config C4 --mode tac --K 2 --B 16"; do
  timeout 600 python bench.py --train --steps 5 --warmup 3 $args 2>&1 | tail -1 | tee -a gpurun_out/train_bench.jsonl
done
