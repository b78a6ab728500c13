for rep in 1 2; do for v in libtacsnn.so libtacsnn_nopack.so; do
  for c in "C2 0 tac 4" "C3 0 tac 8" "C2 0 dense 1"; do set -- $c
    t=$(TACSNN_LIB=paper_2603_13810_b200/$v python scripts/profile_layer.py --config $1 --layer $2 --mode $3 --K $4 --B 1024 --iters 6 2>&1 | grep " ms " | tail -2 | awk '{print $1}' | tr '\n' ' ')
    echo "rep $rep $v $c: $t"
  done; done; done
