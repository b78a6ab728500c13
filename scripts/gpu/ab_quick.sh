# quick parity subset + A/B of the current library against variant libraries (args)
python -m paper_2603_13810_b200.build > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests -x -q -m gpu -k "layer_parity or reset_variants or chaining or config_stack or exhaustive" > gpurun_out/pytest_q.log 2>&1; echo "pytest_rc=$?"; tail -2 gpurun_out/pytest_q.log
bash scripts/gpu/ab_vars.sh libtacsnn.so "$@"
