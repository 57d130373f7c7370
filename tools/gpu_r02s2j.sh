out=gpurun_out/s2j; mkdir -p $out
timeout 600 python -m pytest tests/test_gpu_sessions.py -x -q > $out/pytest.txt 2>&1; echo "exit $?" >> $out/pytest.txt
timeout 900 python tools/ab_sessions.py --workload c1 --rounds 9 --steps 40 --variants "fin1:;fin2:FL_GLM_SOLO_FIN=2" > $out/ab_c1.txt 2>&1
tail -3 $out/pytest.txt; cat $out/ab_c1.txt | grep c1
