# A/B of variant libraries ($LIBS) on the dominant C5 layers and the rate-coded first layers, round robin x2
for rep in 1 2; do
  for c in "C5 0 tactp 4 2048" "C5 1 tactp 4 512" "C3 0 tac 8 1024" "C3 1 tac 8 1024" "C2 0 tac 4 256"; do set -- $c
    for v in $LIBS; do
      t=$(TACSNN_LIB=paper_2603_13810_b200/$v python scripts/profile_layer.py --config $1 --layer $2 --mode $3 --K $4 --B $5 --iters 6 --no-counts 2>&1 | grep " ms " | tail -3 | awk '{print $1}' | tr '\n' ' ')
      echo "rep $rep $c $v: $t"
    done
  done
done
