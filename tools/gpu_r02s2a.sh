out=gpurun_out/s2a; mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $out/smi.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.txt 2>&1; echo "exit $?" >> $out/smoke.txt
timeout 2400 python -m pytest tests -m gpu -x -q > $out/pytest.txt 2>&1; echo "exit $?" >> $out/pytest.txt
timeout 900 python bench.py > $out/bench_c2.json 2> $out/bench_c2.err
timeout 600 python bench.py --workload c3 --no-cpu > $out/bench_c3.json 2> $out/bench_c3.err
tail -3 $out/smoke.txt $out/pytest.txt; cut -c1-400 $out/bench_c2.json $out/bench_c3.json
