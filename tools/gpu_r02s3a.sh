out=gpurun_out/s3a; mkdir -p $out
timeout 1200 python -m pytest tests -m gpu -x -q > $out/pytest_gpu.txt 2>&1; echo "exit $?" >> $out/pytest_gpu.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.txt 2>&1; echo "exit $?" >> $out/smoke.txt
timeout 900 python bench.py > $out/bench_c2.json 2> $out/bench_c2.err
timeout 600 python bench.py --workload c4 --no-cpu > $out/bench_c4.json 2> $out/bench_c4.err
tail -2 $out/pytest_gpu.txt; tail -2 $out/smoke.txt; cut -c1-300 $out/bench_c2.json; cut -c1-200 $out/bench_c4.json
