out=gpurun_out/s3h; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_trainers.py tests/test_gpu_configs.py tests/test_gpu_generic.py tests/test_gpu_nccl.py tests/test_gpu_edge.py -x -q -k "kmeans or KMeans or km or nccl" > $out/pytest.txt 2>&1; echo "exit $?" >> $out/pytest.txt
timeout 900 python tools/ab_sessions.py --workload c3 --rounds 5 --steps 50 --variants "split2:;split1:FL_KM_DIME_SPLIT=1" > $out/ab.txt 2>&1
tail -2 $out/pytest.txt; grep -E "^c3" $out/ab.txt | cut -c1-200
