# A/B of the waiting-role knobs (TACSNN_SLEEP_NS x TACSNN_REFILL_EARLY) on the C5 layers for K = 2, 4, 8
for rep in 1 2; do
  for c in "1 2048 4" "1 2048 8" "1 2048 2" "2 2048 8" "0 1024 2" "0 1024 8"; do set -- $c
    for knobs in "0 1" "512 1" "0 0" "512 0"; do set -- $c $knobs
      t=$(TACSNN_SLEEP_NS=$4 TACSNN_REFILL_EARLY=$5 python scripts/profile_layer.py --config C5 --layer $1 --B $2 --mode tactp --K $3 --iters 3 --no-counts 2>&1 | grep " ms " | tail -2 | awk '{print $1}' | tr '\n' ' ')
      echo "rep $rep C5 L$1 K=$3 sleep=$4 early=$5: $t"
    done
  done
done
