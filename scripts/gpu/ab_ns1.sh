# A/B of variant libraries ($LIBS) on the NS <= 2 (TAC / dense) layers: first layers by graph replay, C5 L0/L1 TAC, C4 L0
for rep in 1 2; do
  for c in "C3 0 tac 8 1024" "C3 1 tac 8 1024" "C2 0 tac 4 256" "C2 1 tac 4 256" "C3 0 dense 1 1024"; do set -- $c
    for v in $LIBS; do
      t=$(TACSNN_LIB=paper_2603_13810_b200/$v python scripts/graph_layer.py --config $1 --layer $2 --mode $3 --K $4 --B $5 2>&1 | grep "graph us" | sed 's/.*launch: //')
      echo "rep $rep $c $v: $t"
    done
  done
  for c in "C5 0 tac 4 1024" "C5 1 tac 4 1024" "C5 0 dense 1 512" "C4 0 tactp 2 64"; do set -- $c
    for v in $LIBS; do
      t=$(TACSNN_LIB=paper_2603_13810_b200/$v python scripts/profile_layer.py --config $1 --layer $2 --mode $3 --K $4 --B $5 --iters 3 --no-counts 2>&1 | grep " ms " | tail -2 | awk '{print $1}' | tr '\n' ' ')
      echo "rep $rep $c $v: $t"
    done
  done
done
