out=gpurun_out/r02v; mkdir -p $out
timeout 600 python -m pytest tests/test_gpu_ops.py -q -k "crossprod" > $out/pytest_cp.txt 2>&1
echo "exit $?" >> $out/pytest_cp.txt
timeout 900 python tools/op_probe.py --crossprod c2 > $out/op_crossprod.txt 2>&1
FL_BENCH_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --workload c1 --steps 5 --warmup 3 --no-cpu > $out/bench_gloo2_c1.json 2> $out/bench_gloo2_c1.err
