#!/bin/bash
# A/B the table-kernel experiment switches (device-resident cfg2)
for cfg in "1 8" "1 12" "1 16" "0 16"; do set -- $cfg
  for n in 10000 40000; do
    echo -n "V=$1 NW=$2 "; BPLB_TAB_V=$1 BPLB_TAB_NW=$2 python scripts/profile_batch.py --nodes $n --reps 6 | tail -1
  done
done
