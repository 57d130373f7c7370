out=gpurun_out/s2k; mkdir -p $out
L=paper_2502_01985_b200/_lib
cp $L/libfl_b200.so /tmp/libfl_cur.so
timeout 600 python -m pytest tests/test_gpu_t5.py tests/test_gpu_trainers.py tests/test_gpu_configs.py -x -q -k "gnmf or GNMF or t5 or c4" > $out/pytest.txt 2>&1; echo "exit $?" >> $out/pytest.txt
for rep in 1 2; do
  cp /tmp/libfl_cur.so $L/libfl_b200.so
  timeout 600 python tools/ab_sessions.py --workload c4 --rounds 3 --steps 10 --variants "early:" >> $out/ab.txt 2>&1
  cp $L/libfl_b200_alt.so $L/libfl_b200.so
  timeout 600 python tools/ab_sessions.py --workload c4 --rounds 3 --steps 10 --variants "late:" >> $out/ab.txt 2>&1
done
cp /tmp/libfl_cur.so $L/libfl_b200.so
tail -2 $out/pytest.txt; grep -E "^c[0-9]" $out/ab.txt
