out=gpurun_out/r02zj; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_ops.py -q -x -k "crossprod" > $out/pytest_ops.txt 2>&1
echo "exit $?" >> $out/pytest_ops.txt
timeout 900 python tools/op_probe.py --crossprod c2 > $out/op_crossprod.txt 2>&1
timeout 900 ncu --clock-control none --metrics gpu__time_duration.sum --csv --log-file $out/launches_crossprod.csv python tools/op_probe.py --crossprod c2 > /dev/null 2>&1
cat $out/pytest_ops.txt | tail -3; cat $out/op_crossprod.txt | grep -v Warn
