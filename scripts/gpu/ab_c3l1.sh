for rep in 1 2 3; do for v in $LIBS; do
  t=$(TACSNN_LIB=paper_2603_13810_b200/$v python scripts/profile_layer.py --config C3 --layer 1 --mode tac --K 8 --B 1024 --iters 20 --no-counts 2>&1 | grep " ms " | tail -5 | awk '{print $1}' | tr '\n' ' ')
  echo "rep $rep C3 L1 $v: $t"
done; done
