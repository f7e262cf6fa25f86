#!/bin/bash
# 8-way shard times: builds x (default | SIMBA_R0_UP=13 SIMBA_GUIDE=2)
for v in sg4 dpw32 spg0 spg2 dpw32spg2; do
  echo "== $v default: $(bash scripts/shards8_ab.sh $v | tail -1)"
  echo "== $v r0up13 g2: $(SIMBA_R0_UP=13 SIMBA_GUIDE=2 bash scripts/shards8_ab.sh $v | tail -1)"
done
