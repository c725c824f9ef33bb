G2="256 27 96 5 1 2 256"; G3="256 13 256 3 1 1 384"; G4="256 13 384 3 1 1 384"; G5="256 13 384 3 1 1 256"; G1="256 57 64 3 1 0 96"
for g in "$G1" "$G2" "$G3" "$G4" "$G5"; do
  for e in X=1 OMNI_WGRAD_BKT=32 OMNI_FORCE_BN=128 OMNI_FORCE_BN=256 OMNI_FORCE_BN=64 "OMNI_FORCE_SPLITS=4" "OMNI_FORCE_SPLITS=8" "OMNI_FORCE_SPLITS=16" "OMNI_FORCE_SPLITS=32"; do
    echo "$e | $(env $e python tools/conv_probe.py wgrad $g 10 2>&1 | tail -1)"
  done
done
