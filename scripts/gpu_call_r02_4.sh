timeout 900 python -m pytest tests/test_xbest.py tests/test_production_paths.py -q > gpurun_out/c4_tests.log 2>&1; tail -3 gpurun_out/c4_tests.log
echo "== shapes default"; timeout 300 python scripts/probe_shapes.py 0:0 0:8
echo "== shapes row1 depth 1"; SIMBA_LIB=$PWD/paper_2605_08243_b200/_lib/libsimba_row1d1.so timeout 300 python scripts/probe_shapes.py 0:0
echo "== tts"; timeout 600 python scripts/probe_tts.py s12_k4_i08 s12_k4_i37 s12_k4_i09 s13_k4_i04 s13_k4_i03 s11_k4_i02
echo "== stats"; SIMBA_LIB=$PWD/paper_2605_08243_b200/_lib/libsimba_stats.so timeout 300 python scripts/probe_shard_stats.py
echo "== sanitize"; timeout 1500 bash scripts/sanitize.sh
