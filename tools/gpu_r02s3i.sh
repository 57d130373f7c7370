out=gpurun_out/s3i; mkdir -p $out
timeout 900 python tools/op_probe.py --crossprod c2 > $out/op_crossprod.txt 2>&1
OP_KS=8,16,32 timeout 900 python tools/op_probe.py --wide c2 > $out/op_wide.txt 2>&1
grep -v Warn $out/op_crossprod.txt | tail -5; grep -v Warn $out/op_wide.txt | tail -6
