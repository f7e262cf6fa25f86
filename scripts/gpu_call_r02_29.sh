for lib in libsimba_v1.so libsimba_v2.so libsimba_v3.so libsimba_head.so; do for st in 1 0; do
  echo "== $lib STEAL=$st"; SIMBA_STEAL=$st SIMBA_LIB=$PWD/paper_2605_08243_b200/_lib/$lib timeout 300 python scripts/probe_variance.py 20; SIMBA_STEAL=$st SIMBA_LIB=$PWD/paper_2605_08243_b200/_lib/$lib timeout 300 python scripts/probe_shapes.py 0:0
done; done
