out=gpurun_out/r02m; mkdir -p $out
timeout 600 python -m pytest tests/test_gpu_t5.py -q -k gnmf > $out/pytest_g5.txt 2>&1
echo "exit $?" >> $out/pytest_g5.txt
FL_GN_T5=1 timeout 600 python bench.py --workload c4 --no-e2e --no-cpu --no-parity > $out/bench_c4_t5.json 2> $out/bench_c4_t5.err
timeout 600 python bench.py --workload c1 --no-e2e --no-cpu --no-parity > $out/bench_c1.json 2> $out/bench_c1.err
timeout 600 python bench.py --workload c2 --no-e2e --no-cpu --no-parity --no-materialized > $out/bench_c2.json 2> $out/bench_c2.err
timeout 900 ncu --clock-control none --set full --import-source on -k regex:k_glm_fact_w -s 6 -c 1 -o $out/full_c1_solo \
  python bench.py --workload c1 --steps 3 --warmup 3 --no-e2e --no-cpu --no-parity --no-materialized > /dev/null 2>&1
timeout 900 ncu --clock-control none --metrics gpu__time_duration.sum -c 60 --csv --log-file $out/launches_c1.csv \
  python bench.py --workload c1 --steps 5 --warmup 3 --no-e2e --no-cpu --no-parity --no-materialized > /dev/null 2>&1
FL_GLM_SOLO=0 timeout 900 ncu --clock-control none --metrics gpu__time_duration.sum -c 60 --csv --log-file $out/launches_c1_nosolo.csv \
  python bench.py --workload c1 --steps 5 --warmup 3 --no-e2e --no-cpu --no-parity --no-materialized > /dev/null 2>&1
