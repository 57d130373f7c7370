out=gpurun_out/r02q; mkdir -p $out
timeout 600 python -m pytest tests/test_gpu_ops.py -q -k "tcgen05 or narrow_lmm or operators" > $out/pytest_ops.txt 2>&1
echo "exit $?" >> $out/pytest_ops.txt
timeout 900 python tools/op_probe.py --wide c2 > $out/op_wide_t5.txt 2>&1
timeout 900 ncu --clock-control none --metrics gpu__time_duration.sum --csv --log-file $out/launches_crossprod.csv \
  python tools/op_probe.py --crossprod c2 > /dev/null 2>&1
