out=gpurun_out/s3k; mkdir -p $out
L=paper_2502_01985_b200/_lib
cp $L/libfl_b200.so /tmp/libfl_cur.so
timeout 900 python -m pytest tests/test_gpu_ops.py -x -q -k "rmm or wide or transpose or tlmm" > $out/pytest.txt 2>&1; echo "exit $?" >> $out/pytest.txt
for rep in 1 2; do
  cp /tmp/libfl_cur.so $L/libfl_b200.so
  echo new >> $out/op.txt; OP_KS=8,32 timeout 900 python tools/op_probe.py --wide c2 2>&1 | grep "^k " >> $out/op.txt
  cp $L/libfl_b200_alt.so $L/libfl_b200.so
  echo old >> $out/op.txt; OP_KS=8,32 timeout 900 python tools/op_probe.py --wide c2 2>&1 | grep "^k " >> $out/op.txt
done
cp /tmp/libfl_cur.so $L/libfl_b200.so
tail -2 $out/pytest.txt; cat $out/op.txt
