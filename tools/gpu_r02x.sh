out=gpurun_out/r02x; mkdir -p $out
timeout 600 python -m pytest tests/test_gpu_ops.py -q -k "crossprod" > $out/pytest.txt 2>&1
echo "exit $?" >> $out/pytest.txt
timeout 900 python tools/op_probe.py --crossprod c2 > $out/op_crossprod.txt 2>&1
for dg in 0 1 2 3; do
  FL_KM_DIAG=$dg timeout 600 python bench.py --workload c3 --steps 30 --no-e2e --no-cpu --no-parity > $out/bench_c3_diag$dg.json 2> $out/bench_c3_diag$dg.err
done
timeout 600 ncu --clock-control none --set full --import-source on -k regex:k_fgram_t5 -s 1 -c 1 -o $out/full_fgram python tools/op_probe.py --crossprod c2 > /dev/null 2>&1
ls -la $out
