out=gpurun_out/r02zn; mkdir -p $out
timeout 300 python tools/tc_probe.py timing > $out/tc_timing.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_ops.py tests/test_gpu_t5.py -q -x -k "crossprod or wide or transpose or rmm or gnmf or random_star" > $out/pytest.txt 2>&1
echo "exit $?" >> $out/pytest.txt
timeout 900 python tools/op_probe.py --crossprod c2 > $out/op_crossprod.txt 2>&1
OP_KS=8,16,32 timeout 900 python tools/op_probe.py --wide c2 > $out/op_wide.txt 2>&1
timeout 900 python bench.py --workload c4 --steps 20 --no-e2e --no-cpu --no-parity > $out/bench_c4.json 2> $out/bench_c4.err
head -3 $out/tc_timing.txt; tail -3 $out/pytest.txt; cat $out/op_*.txt | grep -v Warn
python -c "import json; d=json.loads(open('$out/bench_c4.json').read().strip().splitlines()[-1]); print('c4', d['value'], d['roofline']['kernel_ms'], d['roofline']['frac'])"
