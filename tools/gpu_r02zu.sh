out=gpurun_out/r02zu; mkdir -p $out
timeout 1200 python -m pytest tests/test_gpu_trainers.py tests/test_gpu_configs.py -q -x > $out/pytest.txt 2>&1
echo "exit $?" >> $out/pytest.txt
for w in c1 c2 c3; do
  timeout 900 python bench.py --workload $w --no-e2e --no-cpu --no-parity > $out/bench_$w.json 2> $out/bench_$w.err
done
tail -2 $out/pytest.txt
for w in c1 c2 c3; do python -c "import json; d=json.loads(open('$out/bench_$w.json').read().strip().splitlines()[-1]); print('$w', d['value'], d['roofline']['kernel_ms'], d['roofline']['frac'])"; done
