out=gpurun_out/r02zh; mkdir -p $out
timeout 900 python tools/op_probe.py --crossprod c2 > $out/op_crossprod.txt 2>&1
OP_KS=8,16,32 timeout 900 python tools/op_probe.py --wide c2 > $out/op_wide.txt 2>&1
cat $out/*.txt | grep -v Warn
