out=gpurun_out/s2z; mkdir -p $out
L=paper_2502_01985_b200/_lib
cp $L/libfl_b200.so /tmp/libfl_cur.so
timeout 600 python -m pytest tests/test_gpu_t5.py -x -q > $out/pytest.txt 2>&1; echo "exit $?" >> $out/pytest.txt
for rep in 1 2; do
  cp /tmp/libfl_cur.so $L/libfl_b200.so
  timeout 600 python tools/ab_sessions.py --workload c4 --rounds 3 --steps 10 --variants "nreg112:" >> $out/ab.txt 2>&1
  cp $L/libfl_b200_alt.so $L/libfl_b200.so
  timeout 600 python tools/ab_sessions.py --workload c4 --rounds 3 --steps 10 --variants "reg96:" >> $out/ab.txt 2>&1
done
cp /tmp/libfl_cur.so $L/libfl_b200.so
tail -2 $out/pytest.txt; grep -E "^c4" $out/ab.txt | cut -c1-100
