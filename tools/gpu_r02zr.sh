out=gpurun_out/r02zr; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_ops.py -q -x -k "crossprod" > $out/pytest.txt 2>&1
echo "exit $?" >> $out/pytest.txt
timeout 900 python tools/op_probe.py --crossprod c2 > $out/op_crossprod.txt 2>&1
timeout 900 ncu --clock-control none --metrics gpu__time_duration.sum --csv --log-file $out/launches.csv python tools/op_probe.py --crossprod c2 > /dev/null 2>&1
tail -2 $out/pytest.txt; grep -v Warn $out/op_crossprod.txt
