# A/B: RF-tile column prefetch; shard claim guide / R0+1 row condition
for lib in libsimba.so libsimba_nopf.so libsimba.so libsimba_nopf.so; do
  echo "== $lib"; SIMBA_LIB=$PWD/paper_2605_08243_b200/_lib/$lib timeout 300 python scripts/probe_shapes.py 0:0
done
for cfg in "SIMBA_GUIDE=1" "SIMBA_GUIDE=2" "SIMBA_GUIDE=2 SIMBA_R0_ROWS=8" "SIMBA_GUIDE=1 SIMBA_FINE_ROW=0"; do
  echo "== $cfg"; env $cfg timeout 300 python scripts/probe_shapes.py 0:0
done
