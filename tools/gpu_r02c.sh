out=gpurun_out/r02c; mkdir -p $out
timeout 300 python tools/tc_probe.py > $out/tc_probe.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_generic.py tests/test_gpu_nccl.py -q > $out/pytest_new.txt 2>&1
echo "exit $?" >> $out/pytest_new.txt
