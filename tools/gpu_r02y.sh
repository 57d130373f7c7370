out=gpurun_out/r02y; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_ops.py -q -x > $out/pytest_ops.txt 2>&1
echo "exit $?" >> $out/pytest_ops.txt
OP_KS=3,8,16,32 timeout 900 python tools/op_probe.py --wide c2 > $out/op_wide.txt 2>&1
FL_NO_TMM_T5=1 OP_KS=3,16 timeout 900 python tools/op_probe.py --wide c2 > $out/op_wide_old.txt 2>&1
timeout 600 python tools/scatter_probe.py > $out/scatter.txt 2>&1
OP_KS=32 timeout 900 ncu --clock-control none --metrics gpu__time_duration.sum --csv --log-file $out/launches_wide32.csv python tools/op_probe.py --wide c2 > /dev/null 2>&1
OP_KS=32 timeout 900 ncu --clock-control none --set full --import-source on -k regex:k_tmm_t5 -c 1 -o $out/full_tmm_t5 python tools/op_probe.py --wide c2 > /dev/null 2>&1
ls -la $out
