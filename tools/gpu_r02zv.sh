out=gpurun_out/r02zv; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_ops.py -q -x -k "wide or transpose or rmm or random_star or spec or operators" > $out/pytest.txt 2>&1
echo "exit $?" >> $out/pytest.txt
OP_KS=8,16,32 timeout 900 python tools/op_probe.py --wide c2 > $out/op_wide.txt 2>&1
FL_TMM_YD=1 OP_KS=32 timeout 900 python tools/op_probe.py --wide c2 > $out/op_wide_yd.txt 2>&1
OP_KS=32 timeout 900 ncu --clock-control none --metrics gpu__time_duration.sum --csv --log-file $out/launches.csv python tools/op_probe.py --wide c2 > /dev/null 2>&1
tail -2 $out/pytest.txt; grep -v Warn $out/op_wide.txt $out/op_wide_yd.txt
