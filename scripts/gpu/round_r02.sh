# round-2 evidence refresh: full GPU suite, sweep, bench line, training bench
bash scripts/gpu/tests.sh
timeout 1500 python scripts/sweep.py --out gpurun_out/sweep_r02.jsonl > gpurun_out/sweep.log 2>&1; echo "sweep_rc=$?"
timeout 600 python bench.py > gpurun_out/bench_r02.json 2> gpurun_out/bench.err; echo "bench_rc=$?"; tail -c 300 gpurun_out/bench_r02.json
rm -f gpurun_out/train_bench_r02.jsonl
for args in "--config C4 --mode tactp --K 2 --B 16" "--config C4 --mode tac --K 2 --B 16" "--config C3 --mode tac --K 8" "--config C3 --mode tac --K 8 --whole-net" "--config C2 --mode tac --K 4 --whole-net"; do
  timeout 600 python bench.py --train --steps 5 --warmup 2 $args 2>&1 | tail -1 >> gpurun_out/train_bench_r02.jsonl
done
tail -5 gpurun_out/train_bench_r02.jsonl | cut -c1-200
