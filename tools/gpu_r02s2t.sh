out=gpurun_out/s2t; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_sessions.py tests/test_gpu_trainers.py -x -q -k "staged or gnmf or sessions" > $out/pytest.txt 2>&1; echo "exit $?" >> $out/pytest.txt
timeout 900 python tools/e2e_c4_probe.py --public --jobs 1 > $out/public.txt 2>&1
FL_NO_STAGED_COPY=1 timeout 900 python tools/e2e_c4_probe.py --public --jobs 1 > $out/public_nostage.txt 2>&1
tail -2 $out/pytest.txt; tail -1 $out/public.txt; tail -1 $out/public_nostage.txt
