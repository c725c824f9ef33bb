# weight-gradient GEMMs of CaffeNet conv2-5 on CTA pairs: stage depth and tile width
for L in "256 27 96 5 1 2 256" "256 13 256 3 1 1 384" "256 13 384 3 1 1 384" "256 13 384 3 1 1 256"; do
  for e in X=1 OMNI_WGRAD_BKT=32 OMNI_FORCE_BN=256 OMNI_FORCE_BN=128 "OMNI_FORCE_BN=256 OMNI_WGRAD_BKT=32"; do
    echo "$e | $(env $e python tools/conv_probe.py wgrad $L 10 2>&1 | tail -1)"
  done
done
