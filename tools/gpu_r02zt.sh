out=gpurun_out/r02zt; mkdir -p $out
timeout 1200 python -m pytest tests/test_gpu_t5.py tests/test_gpu_trainers.py tests/test_gpu_generic.py tests/test_gpu_config_parity.py -q -x -k "gnmf or GNMF or nmf" > $out/pytest.txt 2>&1
echo "exit $?" >> $out/pytest.txt
timeout 900 python bench.py --workload c4 --steps 20 --no-e2e --no-cpu --no-parity > $out/bench_c4.json 2> $out/bench_c4.err
tail -3 $out/pytest.txt
python -c "import json; d=json.loads(open('$out/bench_c4.json').read().strip().splitlines()[-1]); print('c4', d['value'], d['roofline']['kernel_ms'], d['roofline']['frac'])"
tail -3 $out/bench_c4.err
