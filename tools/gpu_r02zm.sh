out=gpurun_out/r02zm; mkdir -p $out
timeout 300 python tools/tc_probe.py timing > $out/tc_timing.txt 2>&1
OP_KS=8,16,32 timeout 900 python tools/op_probe.py --wide c2 > $out/op_wide.txt 2>&1
tail -4 $out/tc_timing.txt; cat $out/op_wide.txt | grep -v Warn
