python -m paper_2603_13810_b200.build > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -x -q -m gpu -k "mnist or C2 or C3 or C1 or T25 or agg_weights or runtime_group or prescale or exhaustive or split or real_input" > gpurun_out/pytest_q.log 2>&1; echo "pytest_rc=$?"; tail -3 gpurun_out/pytest_q.log
LIBS="libtacsnn.so libtacsnn_prev.so" bash scripts/gpu/ab_first.sh
