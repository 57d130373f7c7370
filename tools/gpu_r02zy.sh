out=gpurun_out/r02zy; mkdir -p $out
for m in 2 3; do
FL_LMM_T5=$m OP_KS=32 timeout 900 ncu --clock-control none --metrics gpu__time_duration.sum --csv --log-file $out/launches_$m.csv python tools/op_probe.py --wide c2 > /dev/null 2>&1
done
