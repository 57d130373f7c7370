out=gpurun_out/s2e; mkdir -p $out
timeout 600 python -m pytest tests/test_gpu_sessions.py -x -q > $out/pytest_sessions.txt 2>&1; echo "exit $?" >> $out/pytest_sessions.txt
timeout 900 python tools/ab_sessions.py --workload c1 --rounds 7 --steps 40 --variants "new:;red1:FL_GLM_SOLO_RED=1;nos0:FL_GLM_SOLO_S0=0;old:FL_GLM_SOLO_RED=1,FL_GLM_SOLO_S0=0;three:FL_GLM_SOLO=0" > $out/ab_c1.txt 2>&1
tail -3 $out/pytest_sessions.txt; tail -8 $out/ab_c1.txt
