out=gpurun_out/r02l; mkdir -p $out
timeout 600 python -m pytest tests/test_gpu_t5.py -q -k gnmf > $out/pytest_g5.txt 2>&1
echo "exit $?" >> $out/pytest_g5.txt
timeout 600 python -m pytest tests/test_gpu_trainers.py -q -k "solo or glm" > $out/pytest_glm.txt 2>&1
echo "exit $?" >> $out/pytest_glm.txt
FL_GN_T5=1 timeout 600 python bench.py --workload c4 --no-e2e --no-cpu --no-parity > $out/bench_c4_t5.json 2> $out/bench_c4_t5.err
timeout 600 python bench.py --workload c1 --no-e2e --no-cpu --no-parity > $out/bench_c1.json 2> $out/bench_c1.err
timeout 600 python bench.py --workload c2 --no-e2e --no-cpu --no-parity --no-materialized > $out/bench_c2.json 2> $out/bench_c2.err
FL_GN_T5=1 timeout 900 ncu --clock-control none --set full --import-source on -k regex:k_gnmf_t5 -s 4 -c 1 -o $out/full_c4_t5 \
  python bench.py --workload c4 --steps 3 --warmup 3 --no-e2e --no-cpu --no-parity > /dev/null 2>&1
