out=gpurun_out/r02i; mkdir -p $out
timeout 600 python -m pytest tests/test_gpu_t5.py -q > $out/pytest_t5.txt 2>&1
echo "exit $?" >> $out/pytest_t5.txt
FL_GN_T5=1 timeout 600 python bench.py --workload c4 --no-e2e --no-cpu --no-parity > $out/bench_c4_t5.json 2> $out/bench_c4_t5.err
FL_KM_T5=1 timeout 600 python bench.py --workload c3 --no-e2e --no-cpu --no-parity > $out/bench_c3_t5.json 2> $out/bench_c3_t5.err
FL_GN_T5=1 timeout 900 ncu --clock-control none --set full --import-source on -k regex:k_gnmf_t5 -s 4 -c 1 -o $out/full_c4_t5 \
  python bench.py --workload c4 --steps 3 --warmup 3 --no-e2e --no-cpu --no-parity > /dev/null 2>&1
