bash scripts/gpu/trace.sh "C3 0 tac 8 1024" "C3 0 dense 1 1024" "C2 0 tac 4 256"
python -m paper_2603_13810_b200.build > /dev/null 2>&1
timeout 600 python -m pytest tests -x -q -m gpu -k "stack or whole or fc_engines" > gpurun_out/pytest_s.log 2>&1; echo "pytest_rc=$?"; tail -3 gpurun_out/pytest_s.log
