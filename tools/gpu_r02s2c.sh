out=gpurun_out/s2c; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_trainers.py tests/test_gpu_configs.py tests/test_gpu_t5.py -x -q > $out/pytest.txt 2>&1; echo "exit $?" >> $out/pytest.txt
timeout 600 python bench.py --workload c1 --no-cpu > $out/c1.json 2> $out/c1.err
FL_GLM_SOLO_S0=0 timeout 600 python bench.py --workload c1 --no-cpu --no-e2e --no-parity > $out/c1_nos0.json 2> $out/c1_nos0.err
timeout 600 python bench.py --workload c3 --no-cpu --no-e2e > $out/c3.json 2> $out/c3.err
timeout 600 python bench.py --workload c4 --no-cpu --no-e2e > $out/c4.json 2> $out/c4.err
tail -2 $out/pytest.txt
for f in $out/c*.json; do python -c "
import json,sys
d=json.load(open('$f')); print('$f', round(d['value'],1), d['ms_per_step'], d['iteration']['kernel_ms'], d['roofline']['frac'], (d.get('e2e') or {}).get('value'), (d.get('parity') or {}).get('ok'))"; done
