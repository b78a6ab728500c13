# full GPU test suite (+ optional -k filter in $1)
python -m paper_2603_13810_b200.build > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
if [ -n "$1" ]; then
  timeout 1500 python -m pytest tests -x -q -m gpu -k "$1" > gpurun_out/pytest.log 2>&1; echo "pytest_rc=$?"
else
  timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/pytest.log 2>&1; echo "pytest_rc=$?"
fi
tail -30 gpurun_out/pytest.log
