#!/bin/bash
# A/B timing of libsimba variants: scripts/ab.sh name1 name2 ... (each _lib/libsimba_<name>.so)
# prints the size-13 C5 sweep time of each, 3 alternating rounds
for r in 1 2 3; do
  for v in "$@"; do
    echo -n "$v round $r: "
    SIMBA_LIB=paper_2605_08243_b200/_lib/libsimba_$v.so python scripts/probe.py 12 13 2>&1 | awk '{printf "%s %s  ", $3, $5}'
    echo
  done
done
