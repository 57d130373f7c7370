out=gpurun_out/r02n; mkdir -p $out
timeout 1800 python -m pytest tests -m gpu -q -x > $out/pytest_gpu.txt 2>&1
echo "exit $?" >> $out/pytest_gpu.txt
timeout 600 python bench.py --workload c1 --no-e2e --no-cpu --no-parity > $out/bench_c1.json 2> $out/bench_c1.err
timeout 600 python bench.py --workload c4 --no-e2e --no-cpu > $out/bench_c4.json 2> $out/bench_c4.err
timeout 900 ncu --clock-control none --metrics gpu__time_duration.sum -c 400 --csv --log-file $out/launches_c1.csv \
  python bench.py --workload c1 --steps 20 --warmup 3 --no-e2e --no-cpu --no-parity --no-materialized > /dev/null 2>&1
