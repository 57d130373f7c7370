out=gpurun_out/r02zx; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_ops.py -q -x -k "wide or transpose or rmm or random_star or spec or operators" > $out/pytest.txt 2>&1
echo "exit $?" >> $out/pytest.txt
OP_KS=8,16,32 timeout 900 python tools/op_probe.py --wide c2 > $out/op_wide.txt 2>&1
tail -2 $out/pytest.txt; grep -v Warn $out/op_wide.txt
