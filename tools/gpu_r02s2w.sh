out=gpurun_out/s2w; mkdir -p $out
timeout 900 python tools/ab_sessions.py --workload c3 --rounds 3 --steps 50 --variants "def:;n2:FL_KM_NST=2;n3:FL_KM_NST=3;n4:FL_KM_NST=4" > $out/ab_c3.txt 2>&1
timeout 900 python tools/ab_sessions.py --workload c2 --rounds 3 --steps 30 --variants "def:;n2:FL_GLM_NST=2;n3:FL_GLM_NST=3;n4:FL_GLM_NST=4" > $out/ab_c2.txt 2>&1
grep -E "^c[0-9]" $out/ab_c3.txt $out/ab_c2.txt | cut -c1-110
