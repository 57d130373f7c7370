out=gpurun_out/s3c; mkdir -p $out
timeout 600 python bench.py --workload c1 > $out/bench_c1.json 2> $out/bench_c1.err
timeout 600 ncu --clock-control none --metrics gpu__time_duration.sum -c 400 --csv --log-file $out/launches_c1.csv python bench.py --workload c1 --steps 3 --warmup 3 --no-e2e --no-cpu --no-parity --no-materialized > /dev/null 2>&1
cut -c1-300 $out/bench_c1.json
