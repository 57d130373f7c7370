out=gpurun_out/s3l; mkdir -p $out
timeout 1200 python -m pytest tests -m gpu -q > $out/pytest_gpu.txt 2>&1; echo "exit $?" >> $out/pytest_gpu.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.txt 2>&1; echo "exit $?" >> $out/smoke.txt
tail -2 $out/pytest_gpu.txt; tail -2 $out/smoke.txt
