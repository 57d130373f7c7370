out=gpurun_out/r02u; mkdir -p $out
timeout 900 ncu --clock-control none --metrics gpu__time_duration.sum --csv --log-file $out/launches_crossprod.csv \
  python tools/op_probe.py --crossprod c2 > /dev/null 2>&1
