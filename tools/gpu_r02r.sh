out=gpurun_out/r02r; mkdir -p $out
timeout 600 python -m pytest tests/test_gpu_ops.py -q -k "crossprod or tcgen05" > $out/pytest_ops.txt 2>&1
echo "exit $?" >> $out/pytest_ops.txt
timeout 900 python tools/op_probe.py --crossprod c2 > $out/op_crossprod.txt 2>&1
FL_NO_GRAM_T5=1 timeout 900 python tools/op_probe.py --crossprod c2 > $out/op_crossprod_simt.txt 2>&1
