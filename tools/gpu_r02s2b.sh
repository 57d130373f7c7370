out=gpurun_out/s2b; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_trainers.py tests/test_gpu_configs.py tests/test_gpu_edge.py tests/test_gpu_nccl.py -x -q > $out/pytest.txt 2>&1; echo "exit $?" >> $out/pytest.txt
for v in clean dirty; do
  FL_BENCH_FLUSH=$v timeout 600 python bench.py --workload c1 --no-cpu > $out/c1_$v.json 2> $out/c1_$v.err
done
FL_GLM_SOLO_S0=0 timeout 600 python bench.py --workload c1 --no-cpu --no-e2e --no-parity > $out/c1_nos0.json 2> $out/c1_nos0.err
timeout 600 ncu --clock-control none --metrics gpu__time_duration.sum -k regex:k_glm_fact_w --csv --log-file $out/launch_c1.csv python bench.py --workload c1 --steps 5 --warmup 3 --no-e2e --no-cpu --no-parity --no-materialized > /dev/null 2>&1
tail -2 $out/pytest.txt
for f in $out/c1_*.json; do python -c "
import json,sys
d=json.load(open('$f')); print('$f', d['value'], d['ms_per_step'], d['iteration']['kernel_ms'], (d.get('e2e') or {}).get('value'), d.get('parity',{}) and d['parity'].get('ok'))"; done
grep k_glm $out/launch_c1.csv | tail -8
