# GPU suite + A/B of the current library against variant libraries (args) on C5 L0/L1
bash scripts/gpu/tests.sh
bash scripts/gpu/ab_vars.sh libtacsnn.so "$@"
