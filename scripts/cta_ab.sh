#!/bin/bash
# CTA start/end spread of the fused sweep vs its shards (libsimba_cta.so = -DSIMBA_CTA_TIMES)
for c in "1 0" "2 0" "8 1" "8 7"; do
  echo "== N shard = $c"
  SIMBA_LIB=paper_2605_08243_b200/_lib/libsimba_cta.so timeout 120 python scripts/probe_cta_times.py $c > gpurun_out/cta_$$.log 2>&1
  grep KERNEL_MS gpurun_out/cta_$$.log; python scripts/cta_times.py gpurun_out/cta_$$.log
done
rm -f gpurun_out/cta_$$.log
