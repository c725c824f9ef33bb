# BN sweep of the CaffeNet 13x13 implicit convs (fprop and the flipped-kernel dgrad)
for L in "fprop 256 13 256 3 1 1 384" "fprop 256 13 384 3 1 1 384" "fprop 256 13 384 3 1 1 256" "fprop 256 13 384 3 1 1 256" "fprop 256 13 256 3 1 1 384"; do
  for e in X=1 OMNI_FORCE_BN=128 OMNI_FORCE_BN=256 OMNI_FORCE_BN=64; do
    echo "$e | $(env $e python tools/conv_probe.py $L 10 2>&1 | tail -1)"
  done
done
