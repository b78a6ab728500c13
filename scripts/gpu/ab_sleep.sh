# A/B of the producer / MMA backoff (TACSNN_SLEEP_NS) on C5 L0 (B=2048) and C5 L1 (B=512)
for rep in 1 2; do
  for ns in 0 64 256 1000; do
    for c in "C5 0 2048" "C5 1 512"; do set -- $c
      t=$(TACSNN_SLEEP_NS=$ns python scripts/profile_layer.py --config $1 --layer $2 --B $3 --iters 4 --no-counts 2>&1 | grep " ms " | tail -2 | awk '{print $1}' | tr '\n' ' ')
      echo "rep $rep sleep $ns $c: $t"
    done
  done
done
