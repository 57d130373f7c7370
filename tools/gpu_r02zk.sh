out=gpurun_out/r02zk; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_ops.py -q -x -k "crossprod or wide or transpose or rmm or random_star or spec or operators" > $out/pytest_ops.txt 2>&1
echo "exit $?" >> $out/pytest_ops.txt
timeout 900 python tools/op_probe.py --crossprod c2 > $out/op_crossprod.txt 2>&1
OP_KS=8,16,32 timeout 900 python tools/op_probe.py --wide c2 > $out/op_wide.txt 2>&1
OP_KS=32 timeout 900 ncu --clock-control none --metrics gpu__time_duration.sum --csv --log-file $out/launches_wide32.csv python tools/op_probe.py --wide c2 > /dev/null 2>&1
timeout 900 ncu --clock-control none --metrics gpu__time_duration.sum --csv --log-file $out/launches_crossprod.csv python tools/op_probe.py --crossprod c2 > /dev/null 2>&1
tail -3 $out/pytest_ops.txt; cat $out/op_*.txt | grep -v Warn
