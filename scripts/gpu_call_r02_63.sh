for cfg in "X=1" "SIMBA_L2_PERSIST=0"; do echo "== $cfg"; env $cfg timeout 300 python scripts/probe_tts.py s12_k4_i08 s11_k4_i10; done
