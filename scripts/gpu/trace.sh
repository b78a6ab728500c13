# role timeline of CTA 0 (trace build as a variant library)
TACSNN_LIB_NAME=libtacsnn_trace.so TACSNN_TRACE=1 python -m paper_2603_13810_b200.build --force > gpurun_out/build_trace.log 2>&1 || { tail -30 gpurun_out/build_trace.log; exit 1; }
export TACSNN_LIB=$PWD/paper_2603_13810_b200/libtacsnn_trace.so
for c in "$@"; do set -- $c
  echo "== $c"; python scripts/trace_layer.py --config $1 --layer $2 --mode $3 --K $4 --B $5 --rows 8 2>&1 | tail -16
done
