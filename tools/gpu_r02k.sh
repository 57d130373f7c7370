out=gpurun_out/r02k; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_t5.py tests/test_gpu_trainers.py tests/test_gpu_configs.py tests/test_gpu_edge.py -q -x > $out/pytest.txt 2>&1
echo "exit $?" >> $out/pytest.txt
FL_GN_T5=1 timeout 600 python bench.py --workload c4 --no-e2e --no-cpu --no-parity > $out/bench_c4_t5.json 2> $out/bench_c4_t5.err
timeout 600 python bench.py --workload c1 --no-e2e --no-cpu --no-parity > $out/bench_c1.json 2> $out/bench_c1.err
timeout 600 python bench.py --workload c2 --no-e2e --no-cpu --no-parity --no-materialized > $out/bench_c2.json 2> $out/bench_c2.err
FL_GLM_SOLO=0 timeout 600 python bench.py --workload c1 --no-e2e --no-cpu --no-parity > $out/bench_c1_nosolo.json 2> $out/bench_c1_nosolo.err
