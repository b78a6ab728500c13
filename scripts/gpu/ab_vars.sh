# A/B of variant libraries on C5 layers 0 and 1 (B=512), round robin x2:
#   bash scripts/gpu/ab_vars.sh libtacsnn.so libtacsnn_x.so ...
for rep in 1 2; do
  for L in 0 1; do
    for v in "$@"; do
      t=$(TACSNN_LIB=paper_2603_13810_b200/$v python scripts/profile_layer.py --config C5 --layer $L --B 512 --iters 5 --no-counts 2>&1 | grep " ms " | tail -3 | awk '{print $1}' | tr '\n' ' ')
      echo "rep $rep L$L $v: $t"
    done
  done
done
