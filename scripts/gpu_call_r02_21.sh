for cfg in "SIMBA_SPLIT_MIN=32768" "SIMBA_SPLIT_MIN=65536" "SIMBA_SPLIT_MIN=131072" "SIMBA_SPLIT_MIN=262144" "SIMBA_SPLIT_MIN=524288"; do echo "== $cfg"; env $cfg timeout 300 python scripts/probe_variance.py 40; done
for lib in libsimba_pg2.so libsimba_pg8.so; do echo "== $lib"; SIMBA_LIB=$PWD/paper_2605_08243_b200/_lib/$lib timeout 300 python scripts/probe_variance.py 40; done
for lib in libsimba_pg2.so libsimba_pg8.so; do echo "== $lib split 131072"; SIMBA_SPLIT_MIN=131072 SIMBA_LIB=$PWD/paper_2605_08243_b200/_lib/$lib timeout 300 python scripts/probe_variance.py 40; done
