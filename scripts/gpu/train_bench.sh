python -m paper_2603_13810_b200.build > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_backward.py -x -q -k trainable > gpurun_out/pytest_train.log 2>&1; echo "pytest_rc=$?"; tail -5 gpurun_out/pytest_train.log
for args in "--config C3 --mode tac --K 8" "--config C3 --mode tac --K 8 --whole-net" "--config C2 --mode tac --K 4 --whole-net" "--config C4 --mode tactp --K 2 --B 16" "--config C4 --mode tac --K 2 --B 16"; do
  timeout 600 python bench.py --train --steps 5 --warmup 2 $args 2>&1 | tail -1 | tee -a gpurun_out/train_bench.jsonl
done
