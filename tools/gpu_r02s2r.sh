out=gpurun_out/s2r; mkdir -p $out
timeout 900 python tools/e2e_c4_probe.py --jobs 3 > $out/e2e_c4.txt 2>&1
cat $out/e2e_c4.txt | tail -4
