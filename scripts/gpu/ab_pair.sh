# A/B of the two-groups-per-iteration epilogue (TACSNN_NO_PAIR_GROUPS) on C5 L0 TAC-TP / TAC / dense, C3, C2
for rep in 1 2; do
  for c in "C5 0 tactp 4 2048" "C5 0 tac 4 1024" "C5 0 dense 1 512" "C5 1 tac 4 1024"; do set -- $c
    for env in 0 1; do
      t=$(TACSNN_NO_PAIR_GROUPS=$env python scripts/profile_layer.py --config $1 --layer $2 --mode $3 --K $4 --B $5 --iters 3 --no-counts 2>&1 | grep " ms " | tail -2 | awk '{print $1}' | tr '\n' ' ')
      echo "rep $rep $c nopair=$env: $t"
    done
  done
  for c in "C3 0 tac 8 1024" "C3 1 tac 8 1024" "C2 0 tac 4 256"; do set -- $c
    for env in 0 1; do
      t=$(TACSNN_NO_PAIR_GROUPS=$env python scripts/graph_layer.py --config $1 --layer $2 --mode $3 --K $4 --B $5 2>&1 | grep "graph us" | sed 's/.*launch: //')
      echo "rep $rep $c nopair=$env: $t"
    done
  done
done
