out=gpurun_out/s2p; mkdir -p $out
timeout 900 python tools/ab_sessions.py --workload c1 --rounds 7 --steps 40 --variants "loop:FL_GLM_SOLO_DIAG=32;noloads:FL_GLM_SOLO_DIAG=64;idlefinal:FL_GLM_SOLO_DIAG=16;nofinal:FL_GLM_SOLO_DIAG=2" > $out/ab_c1.txt 2>&1
grep c1 $out/ab_c1.txt | cut -c1-70
