# A/B of variant libraries ($LIBS) on the int8 (halo-path) layers of C5 (B=2048) and C4 (B=64)
for rep in 1 2; do
  for c in "C5 1 2048 tactp 4" "C5 2 2048 tactp 4" "C5 3 2048 tactp 4" "C4 1 64 tactp 2" "C4 2 64 tactp 2"; do set -- $c
    for v in $LIBS; do
      t=$(TACSNN_LIB=paper_2603_13810_b200/$v python scripts/profile_layer.py --config $1 --layer $2 --B $3 --mode $4 --K $5 --iters 4 --no-counts 2>&1 | grep " ms " | tail -2 | awk '{print $1}' | tr '\n' ' ')
      echo "rep $rep $c $v: $t"
    done
  done
done
