out=gpurun_out/r02zo; mkdir -p $out
timeout 300 python tools/tc_probe.py timing > $out/tc_timing.txt 2>&1
cat $out/tc_timing.txt
