out=gpurun_out/r02zp; mkdir -p $out
timeout 2400 python -m pytest tests -q -m gpu -x > $out/pytest_gpu.txt 2>&1
echo "exit $?" >> $out/pytest_gpu.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.txt 2>&1
echo "exit $?" >> $out/smoke.txt
tail -5 $out/pytest_gpu.txt; tail -3 $out/smoke.txt
