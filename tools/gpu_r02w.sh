out=gpurun_out/r02w; mkdir -p $out
timeout 600 python -m pytest tests/test_gpu_ops.py tests/test_gpu_trainers.py -q -k "crossprod or kmeans" > $out/pytest.txt 2>&1
echo "exit $?" >> $out/pytest.txt
timeout 900 python tools/op_probe.py --crossprod c2 > $out/op_crossprod.txt 2>&1
timeout 600 python bench.py --workload c3 --no-e2e --no-cpu > $out/bench_c3.json 2> $out/bench_c3.err
