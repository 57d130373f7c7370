# round 2: new GPU tests (width-general sessions, NCCL), C3/C4 bench lines,
# source-level ncu of the K-means and GNMF fact passes
out=gpurun_out/r02b; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_generic.py tests/test_gpu_nccl.py -x -q > $out/pytest_new.txt 2>&1
echo "exit $?" >> $out/pytest_new.txt
timeout 600 python bench.py --workload c3 --no-e2e --no-cpu > $out/bench_c3.json 2> $out/bench_c3.err
timeout 600 python bench.py --workload c4 --no-e2e --no-cpu > $out/bench_c4.json 2> $out/bench_c4.err
NCU="ncu --clock-control none"
timeout 900 $NCU --set full --import-source on -k regex:k_km_fact -s 4 -c 1 -o $out/full_c3_fact \
  python bench.py --workload c3 --steps 3 --warmup 3 --no-e2e --no-cpu --no-parity > /dev/null 2>&1
timeout 900 $NCU --set full --import-source on -k regex:k_gnmf_fact -s 4 -c 1 -o $out/full_c4_fact \
  python bench.py --workload c4 --steps 3 --warmup 3 --no-e2e --no-cpu --no-parity > /dev/null 2>&1
ls -la $out
