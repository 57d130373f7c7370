out=gpurun_out/s2f; mkdir -p $out
timeout 600 python -m pytest tests/test_gpu_sessions.py tests/test_gpu_t5.py -x -q > $out/pytest.txt 2>&1; echo "exit $?" >> $out/pytest.txt
timeout 900 python tools/ab_sessions.py --workload c4 --rounds 4 --steps 10 --variants "pre:;nopre:FL_GN5_GPRE=0" > $out/ab_c4.txt 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_km_fact -s 4 -c 1 -o $out/full_c3 python bench.py --workload c3 --steps 3 --warmup 3 --no-e2e --no-cpu --no-parity > /dev/null 2>&1
python tools/ncu_source.py $out/full_c3.ncu-rep 120 inst > $out/km_src_inst.txt 2>&1
python tools/ncu_summary.py report $out/full_c3.ncu-rep > $out/km_summary.txt 2>&1
rm -f $out/full_c3.ncu-rep
tail -3 $out/pytest.txt; cat $out/ab_c4.txt | tail -3; head -30 $out/km_src_inst.txt
