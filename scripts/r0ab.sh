#!/bin/bash
# A/B of libsimba variants x r0[:threads] configs, one process per (lib, config):
#   scripts/r0ab.sh "libs" "configs" "sizes"
for r in 1 2; do
  for v in $1; do
    for c in $2; do
      echo -n "$v $c r$r: "
      SIMBA_LIB=paper_2605_08243_b200/_lib/libsimba_$v.so timeout 300 python scripts/probe_r0.py $c --sizes $3 | awk '{printf "%s %s  ", $3, $5}'
      echo
    done
  done
done
