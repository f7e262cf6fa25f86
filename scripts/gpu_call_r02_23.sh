# per-CTA timelines of 6 launches of the full sweep (one launch per process)
for i in 1 2 3 4 5 6; do
  SIMBA_LIB=$PWD/paper_2605_08243_b200/_lib/libsimba_cta.so timeout 120 python scripts/probe_cta_times.py 1 0 > gpurun_out/c23_cta_$i.txt 2>&1
  grep KERNEL_MS gpurun_out/c23_cta_$i.txt; python scripts/cta_times.py gpurun_out/c23_cta_$i.txt
done
