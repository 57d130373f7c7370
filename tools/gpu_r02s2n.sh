out=gpurun_out/s2n; mkdir -p $out
timeout 900 python tools/ab_sessions.py --workload c1 --rounds 7 --steps 40 --variants "base:;notail:FL_GLM_SOLO_DIAG=1;nofinal:FL_GLM_SOLO_DIAG=2;idlefinal:FL_GLM_SOLO_DIAG=16;noupdate:FL_GLM_SOLO_DIAG=4" > $out/ab_c1.txt 2>&1
grep c1 $out/ab_c1.txt | cut -c1-70
