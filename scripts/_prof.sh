mkdir -p gpurun_out
for t in s2d_minb=6 s2d_minb=1; do
  UCUDNN_TUNE=$t timeout 120 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:s2d \
    python scripts/one_conv.py --layer a1 --op 0 --algo 5 --batch 64 --reps 3 > gpurun_out/s2d_$t.csv 2>&1
done
timeout 900 python -m pytest tests/test_algos_gpu.py -x -q > gpurun_out/t_algos.log 2>&1; echo "rc=$?" >> gpurun_out/t_algos.log
rm -f gpurun_out/db.csv; timeout 900 python bench.py --db gpurun_out/db.csv > gpurun_out/bench.json 2> gpurun_out/bench.err
