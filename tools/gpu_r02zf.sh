out=gpurun_out/r02zf; mkdir -p $out
timeout 300 python tools/tc_probe.py timing > $out/tc_timing.txt 2>&1
cat $out/tc_timing.txt
timeout 900 python -m pytest tests/test_gpu_ops.py -q -x -k "crossprod" > $out/pytest_ops.txt 2>&1
echo "exit $?" >> $out/pytest_ops.txt
timeout 900 python tools/op_probe.py --crossprod c2 > $out/op_crossprod.txt 2>&1
timeout 900 ncu --clock-control none --set full -k regex:k_gram -c 2 -o $out/full_kgram python tools/op_probe.py --crossprod c2 > /dev/null 2>&1
