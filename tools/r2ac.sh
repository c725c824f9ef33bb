# Planner sweep for the conv GEMMs below 650 TFLOP/s: tile width x split count x pairs.
run() { echo "== $1 | $2"; env $1 timeout 60 python tools/conv_probe.py $2 20 2>&1 | tail -1; }
for shape in "wgrad 256 13 256 3 1 1 384" "wgrad 256 13 384 3 1 1 384" "fprop 256 27 256 5 1 2 96" "fprop 256 13 384 3 1 1 384"; do
  run "X=0" "$shape"
  for bn in 128 192 256; do run "OMNI_FORCE_BN=$bn" "$shape"; done
  for sp in 2 3 4 6 8 12; do run "OMNI_FORCE_SPLITS=$sp" "$shape"; done
  run "OMNI_NO_2CTA=1" "$shape"
  run "OMNI_WGRAD_BKT=32" "$shape"
  run "OMNI_KMAJOR_BKT=32" "$shape"
  run "OMNI_NO_TRANSPOSED_FPROP=1" "$shape"
done
