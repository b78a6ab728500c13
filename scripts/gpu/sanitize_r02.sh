python -m paper_2603_13810_b200.build > gpurun_out/build.log 2>&1
timeout 1200 compute-sanitizer --tool memcheck --print-limit 20 python scripts/sanitize.py > gpurun_out/sanitizer_memcheck_r02.log 2>&1; echo "memcheck_rc=$?"; tail -4 gpurun_out/sanitizer_memcheck_r02.log
timeout 1200 compute-sanitizer --tool racecheck --print-limit 20 python scripts/sanitize.py --quick > gpurun_out/sanitizer_racecheck_r02.log 2>&1; echo "racecheck_rc=$?"; tail -4 gpurun_out/sanitizer_racecheck_r02.log
timeout 900 compute-sanitizer --tool synccheck --print-limit 20 python scripts/sanitize.py --quick > gpurun_out/sanitizer_synccheck_r02.log 2>&1; echo "synccheck_rc=$?"; tail -4 gpurun_out/sanitizer_synccheck_r02.log
