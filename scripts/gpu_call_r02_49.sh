for i in 1 2; do for lib in libsimba.so libsimba_desc17.so libsimba_split16.so; do
  echo "== $lib"; SIMBA_LIB=$PWD/paper_2605_08243_b200/_lib/$lib timeout 300 python scripts/probe_variance.py 30; SIMBA_LIB=$PWD/paper_2605_08243_b200/_lib/$lib timeout 300 python scripts/probe_shapes.py 0:0
done; done
