out=gpurun_out/r02zq; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_ops.py -q -x -k "lmm" > $out/pytest.txt 2>&1
echo "exit $?" >> $out/pytest.txt
FL_LMM_T5=2 OP_KS=16,32 timeout 900 python tools/op_probe.py --wide c2 > $out/op_wide_t5_2.txt 2>&1
FL_LMM_T5=1 OP_KS=16,32 timeout 900 python tools/op_probe.py --wide c2 > $out/op_wide_t5_1.txt 2>&1
FL_LMM_T5=2 OP_KS=32 timeout 900 ncu --clock-control none --metrics gpu__time_duration.sum --csv --log-file $out/launches.csv python tools/op_probe.py --wide c2 > /dev/null 2>&1
tail -2 $out/pytest.txt; grep -v Warn $out/op_wide_t5_2.txt $out/op_wide_t5_1.txt
