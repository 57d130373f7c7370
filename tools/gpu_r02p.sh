out=gpurun_out/r02p; mkdir -p $out
timeout 600 python -m pytest tests/test_gpu_ops.py -q -k "tcgen05 or narrow_lmm or operators" > $out/pytest_ops.txt 2>&1
echo "exit $?" >> $out/pytest_ops.txt
timeout 900 python tools/op_probe.py --wide c2 > $out/op_wide_t5.txt 2>&1
FL_NO_LMM_T5=1 OP_KS=32 timeout 900 python tools/op_probe.py --wide c2 > $out/op_wide_not5.txt 2>&1
timeout 900 python tools/op_probe.py --crossprod c2 > $out/op_crossprod.txt 2>&1
