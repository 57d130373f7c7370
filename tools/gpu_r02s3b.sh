out=gpurun_out/s3b; mkdir -p $out
timeout 600 python -m pytest tests/test_gpu_sessions.py tests/test_gpu_trainers.py -x -q -k "glm or sessions or linreg or logreg" > $out/pytest.txt 2>&1; echo "exit $?" >> $out/pytest.txt
timeout 900 python tools/ab_sessions.py --workload c1 --rounds 7 --steps 40 --variants "pref:;nopref:FL_GLM_SOLO_DIAG=256;notail:FL_GLM_SOLO_DIAG=1" > $out/ab_c1.txt 2>&1
tail -2 $out/pytest.txt; grep c1 $out/ab_c1.txt | cut -c1-70
