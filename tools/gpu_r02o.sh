out=gpurun_out/r02o; mkdir -p $out
timeout 600 python bench.py --workload c2 --no-e2e --no-cpu --no-parity --no-materialized > $out/bench_c2.json 2> $out/bench_c2.err
timeout 600 python bench.py --workload c3 --no-e2e --no-cpu --no-parity > $out/bench_c3.json 2> $out/bench_c3.err
timeout 900 ncu --clock-control none --set full --import-source on -k regex:k_glm_fact_w -s 10 -c 1 -o $out/full_c1_solo \
  python bench.py --workload c1 --steps 5 --warmup 3 --no-e2e --no-cpu --no-parity --no-materialized > /dev/null 2>&1
