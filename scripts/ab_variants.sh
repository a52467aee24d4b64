#!/bin/bash
# A/B of attention-kernel build variants on one GPU (diagnostic, not the bench):
# for each library (product first and last, to bracket drift) a short-burst
# probe and 8 s sustained power-capped runs.  Usage:
#   scripts/ab_variants.sh lib1.so lib2.so ...   (product = paper_2412_20501_b200/libtokenring.so)
set -u
PROD=paper_2412_20501_b200/libtokenring.so
for lib in "$PROD" "$@" "$PROD"; do
  echo "== $lib"
  TOKENRING_LIB=$lib timeout 300 python scripts/probe_attn.py --case 0
  TOKENRING_LIB=$lib timeout 300 python scripts/probe_attn.py --case 1
  TOKENRING_LIB=$lib timeout 120 python scripts/power_probe.py attn-full 8
  TOKENRING_LIB=$lib timeout 120 python scripts/power_probe.py attn-causal 8
done
