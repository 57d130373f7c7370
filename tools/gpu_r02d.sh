out=gpurun_out/r02d; mkdir -p $out
timeout 600 python tools/tc_probe.py > $out/tc_probe.txt 2>&1
