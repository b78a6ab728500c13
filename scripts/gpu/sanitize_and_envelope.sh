set -x
python -m paper_2603_13810_b200.build > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "cin64 or cin96 or cout8_int8 or cout16_int8 or cin128_cout96" > gpurun_out/env_tests.log 2>&1; echo "env_rc=$?"
tail -5 gpurun_out/env_tests.log
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python scripts/sanitize.py > gpurun_out/san_memcheck.log 2>&1; echo "memcheck_rc=$?"
tail -8 gpurun_out/san_memcheck.log
timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python scripts/sanitize.py --quick > gpurun_out/san_racecheck.log 2>&1; echo "racecheck_rc=$?"
tail -8 gpurun_out/san_racecheck.log
timeout 600 compute-sanitizer --tool synccheck --print-limit 20 python scripts/sanitize.py --quick > gpurun_out/san_synccheck.log 2>&1; echo "synccheck_rc=$?"
tail -8 gpurun_out/san_synccheck.log
