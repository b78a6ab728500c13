# A/B of variant libraries ($LIBS) on C5 layer 0 at the bench batch (B=2048), round robin x3
for rep in 1 2 3; do
  for v in $LIBS; do
    t=$(TACSNN_LIB=paper_2603_13810_b200/$v python scripts/profile_layer.py --config C5 --layer 0 --B ${B:-2048} --iters 4 --no-counts 2>&1 | grep " ms " | tail -2 | awk '{print $1}' | tr '\n' ' ')
    echo "rep $rep C5 L0 $v: $t"
  done
done
