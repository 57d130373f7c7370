out=gpurun_out/s2s; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_trainers.py tests/test_gpu_configs.py tests/test_gpu_ops.py tests/test_gpu_generic.py -x -q > $out/pytest.txt 2>&1; echo "exit $?" >> $out/pytest.txt
timeout 900 python tools/e2e_c4_probe.py --jobs 3 > $out/e2e_c4.txt 2>&1
FL_NO_STAGED_D2H=1 timeout 900 python tools/e2e_c4_probe.py --jobs 2 > $out/e2e_c4_nostage.txt 2>&1
L=paper_2502_01985_b200/_lib
cp $L/libfl_b200.so /tmp/libfl_cur.so
for rep in 1 2; do
  cp /tmp/libfl_cur.so $L/libfl_b200.so
  timeout 600 python tools/ab_sessions.py --workload c4 --rounds 3 --steps 10 --variants "nowait:" >> $out/ab.txt 2>&1
  cp $L/libfl_b200_alt.so $L/libfl_b200.so
  timeout 600 python tools/ab_sessions.py --workload c4 --rounds 3 --steps 10 --variants "wait:" >> $out/ab.txt 2>&1
done
cp /tmp/libfl_cur.so $L/libfl_b200.so
tail -2 $out/pytest.txt; tail -3 $out/e2e_c4.txt; tail -2 $out/e2e_c4_nostage.txt; grep -E "^c4" $out/ab.txt | cut -c1-70
