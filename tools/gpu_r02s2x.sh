out=gpurun_out/s2x; mkdir -p $out
timeout 900 python tools/ab_sessions.py --workload c4 --rounds 6 --steps 10 --variants "pd6:;pd3:FL_GN5_PD=3;pd0:FL_GN5_PD=0" > $out/ab_c4b.txt 2>&1
grep -E "^c[0-9]" $out/ab_c4b.txt | cut -c1-130
