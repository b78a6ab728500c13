TACSNN_LIB_NAME=libtacsnn_trace.so TACSNN_TRACE=1 python -m paper_2603_13810_b200.build --force > gpurun_out/build_trace.log 2>&1
export TACSNN_LIB=$PWD/paper_2603_13810_b200/libtacsnn_trace.so
python scripts/trace_layer.py --config C3 --layer 0 --mode tac --K 8 --B 1024 --rows 60 2>&1 | tail -75
