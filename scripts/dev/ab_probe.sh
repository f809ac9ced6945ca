#!/bin/bash
# A/B of two libtgv builds on the same box (dev): C4 1024^3 and C2 fused sweep per-launch times.
# usage: ab_probe.sh OUT lib_a lib_b
OUT=$1; A=$2; B=$3
for rep in 1 2; do
  for L in $A $B; do
    TGV_LIB=$L timeout 300 python scripts/dev/c4_probe.py 1024 0 20 2>&1 | grep -v Warn | sed "s|^|$(basename $L) |" >> $OUT
    TGV_LIB=$L timeout 300 python scripts/dev/c4_probe.py 256 0 60 2>&1 | grep -v Warn | sed "s|^|$(basename $L) |" >> $OUT
  done
done
