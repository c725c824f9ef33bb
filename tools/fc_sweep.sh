# Split-count / tile-width sweep of the CaffeNet FC-layer GEMMs (b = 256):
# forward (M = b), weight gradient (K = b) and data gradient, in the operand
# layouts engine.py uses.  One process per setting (the planner reads the
# OMNI_FORCE_* knobs once).  Output: one line per (shape, setting).
for S in "256 4096 9216 0 0" "256 4096 4096 0 0" "256 1000 4096 0 0" \
         "9216 4096 256 1 1" "4096 4096 256 1 1" "4096 1000 256 1 1" \
         "256 9216 4096 0 0" "256 4096 4096 0 0" "256 4096 1000 0 0"; do
  for e in X=1 OMNI_FORCE_SPLITS=1 OMNI_FORCE_SPLITS=2 OMNI_FORCE_SPLITS=3 OMNI_FORCE_SPLITS=4 \
           OMNI_FORCE_SPLITS=6 OMNI_FORCE_SPLITS=8 OMNI_FORCE_SPLITS=12 OMNI_FORCE_SPLITS=16 \
           "OMNI_FORCE_BN=128 OMNI_FORCE_SPLITS=2" "OMNI_FORCE_BN=128 OMNI_FORCE_SPLITS=4" \
           OMNI_FORCE_BN=128 OMNI_NO_2CTA=1; do
    echo "$e | $(env $e python tools/gemm_probe.py $S tf32 20 2>&1 | tail -1)"
  done
done
