# bench + launch list + full captures of the two dominant kernels (run on the GPU box)
R=${1:-r01h}
set -x
timeout 600 python bench.py > gpurun_out/bench_${R}.json 2> gpurun_out/bench_${R}.err
tail -c 600 gpurun_out/bench_${R}.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"select_bits|actquant|qlinear" -c 400 --csv \
  --log-file gpurun_out/launches_${R}.csv python bench.py --steps 2 --warmup 3 --trials 1 --profile --no-cpu --no-prefill > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:qlinear_decode_kernel -s 4 -c 1 \
  -o gpurun_out/${R}_decode_gate_up python tools/prof_decode.py gate_up 8 4 4 > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:qlinear_prefill_kernel -s 2 -c 1 \
  -o gpurun_out/${R}_prefill_gate_up python tools/prof_prefill.py gate_up 288 4 4 > /dev/null 2>&1
ls -la gpurun_out/
for r in ${R}_decode_gate_up ${R}_prefill_gate_up; do
  ncu -i gpurun_out/$r.ncu-rep --page raw --csv > gpurun_out/$r.raw.csv 2>/dev/null
done
