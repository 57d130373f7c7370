out=gpurun_out/s2d; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_trainers.py tests/test_gpu_configs.py tests/test_gpu_edge.py tests/test_gpu_nccl.py -x -q > $out/pytest.txt 2>&1; echo "exit $?" >> $out/pytest.txt
timeout 600 python bench.py --workload c1 --no-cpu > $out/c1.json 2> $out/c1.err
FL_GLM_DIRECT=1 timeout 600 python bench.py --workload c1 --no-cpu --no-e2e --no-parity > $out/c1_direct.json 2> $out/c1_direct.err
FL_TRACE_UPLOAD=1 timeout 900 python bench.py --no-cpu --no-parity --no-materialized > $out/c2.json 2> $out/c2.err
tail -2 $out/pytest.txt
for f in $out/c*.json; do python -c "
import json,sys
d=json.load(open('$f')); print('$f', round(d['value'],1), d['ms_per_step'], d['iteration']['kernel_ms'], d['roofline']['frac'], (d.get('e2e') or {}).get('value'), (d.get('e2e') or {}).get('phases_seconds'), (d.get('parity') or {}).get('ok'))"; done
grep -v "^\s*$" $out/c2.err | tail -40
