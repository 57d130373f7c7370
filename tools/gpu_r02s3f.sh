out=gpurun_out/s3f; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_trainers.py tests/test_gpu_configs.py tests/test_gpu_generic.py tests/test_gpu_nccl.py tests/test_gpu_t5.py tests/test_gpu_distributed.py -x -q -k "kmeans or KMeans or km or nccl or sharded" > $out/pytest.txt 2>&1; echo "exit $?" >> $out/pytest.txt
for rep in 1 2; do
  timeout 600 python tools/ab_sessions.py --workload c3 --rounds 3 --steps 50 --variants "pdl:" >> $out/ab.txt 2>&1
  FL_NO_PDL=1 timeout 600 python tools/ab_sessions.py --workload c3 --rounds 3 --steps 50 --variants "nopdl:" >> $out/ab.txt 2>&1
done
tail -2 $out/pytest.txt; grep -E "^c3" $out/ab.txt | cut -c1-100
