out=gpurun_out/s2g; mkdir -p $out
L=paper_2502_01985_b200/_lib
cp $L/libfl_b200.so /tmp/libfl_cur.so
for rep in 1 2; do
  cp /tmp/libfl_cur.so $L/libfl_b200.so
  timeout 600 python tools/ab_sessions.py --workload c4 --rounds 3 --steps 10 --variants "elect_pre:;elect_nopre:FL_GN5_GPRE=0" >> $out/ab_c4.txt 2>&1
  cp $L/libfl_b200_lane0.so $L/libfl_b200.so
  timeout 600 python tools/ab_sessions.py --workload c4 --rounds 3 --steps 10 --variants "lane0_pre:;lane0_nopre:FL_GN5_GPRE=0" >> $out/ab_c4.txt 2>&1
done
cp /tmp/libfl_cur.so $L/libfl_b200.so
cat $out/ab_c4.txt | grep c4
