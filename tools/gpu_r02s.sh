out=gpurun_out/r02s; mkdir -p $out
timeout 600 python -m pytest tests/test_gpu_ops.py -q -k "crossprod" > $out/pytest_cp.txt 2>&1
echo "exit $?" >> $out/pytest_cp.txt
timeout 900 python tools/op_probe.py --crossprod c2 > $out/op_crossprod.txt 2>&1
timeout 3000 python bench_sweep.py --rows 10000000 --out gpurun_out/r02s/r02_c5_sweep_10M > $out/sweep.log 2>&1
echo "sweep exit $?" >> $out/sweep.log
