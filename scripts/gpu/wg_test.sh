python -m paper_2603_13810_b200.build > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 600 python -m pytest tests/test_gpu_backward.py -x -q -k "dvsL2 and tcgen05" > gpurun_out/pytest_wg0.log 2>&1; echo "noswap_rc=$?"; grep -m3 "Error\|max err" gpurun_out/pytest_wg0.log; tail -2 gpurun_out/pytest_wg0.log
TACSNN_WG_SWAP=1 timeout 600 python -m pytest tests/test_gpu_backward.py -x -q -k "dvsL2 and tcgen05" > gpurun_out/pytest_wg1.log 2>&1; echo "swap_rc=$?"; grep -m3 "Error\|max err" gpurun_out/pytest_wg1.log; tail -2 gpurun_out/pytest_wg1.log
