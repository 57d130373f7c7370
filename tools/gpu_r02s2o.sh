out=gpurun_out/s2o; mkdir -p $out
timeout 600 python -m pytest tests/test_gpu_sessions.py tests/test_gpu_trainers.py tests/test_gpu_configs.py -x -q > $out/pytest.txt 2>&1; echo "exit $?" >> $out/pytest.txt
timeout 900 python tools/ab_sessions.py --workload c1 --rounds 7 --steps 40 --variants "batched:;loop:FL_GLM_SOLO_DIAG=32;idlefinal:FL_GLM_SOLO_DIAG=16" > $out/ab_c1.txt 2>&1
tail -2 $out/pytest.txt; grep c1 $out/ab_c1.txt | cut -c1-70
