# ncu captures + source pages for the decode and prefill kernels (run on the GPU box)
set -x
O=gpurun_out/p
mkdir -p $O
python tools/prof_decode.py gate_up 8 4 4
python tools/prof_decode.py gate_up 8 4 16
DYQ_DEBUG_SKIP=1 python tools/prof_decode.py gate_up 8 4 4
python tools/prof_decode.py o 8 4 4
python tools/prof_decode.py down 8 4 4
timeout 300 ncu --set full --clock-control none --import-source on -k regex:qlinear_decode_kernel -s 4 -c 1 \
  -o $O/dec_a4 python tools/prof_decode.py gate_up 8 4 4 > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:actquant_dec -s 4 -c 1 \
  -o $O/aq python tools/prof_decode.py gate_up 8 4 4 > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:qlinear_prefill_kernel -s 2 -c 1 \
  -o $O/pre_a4 python tools/prof_prefill.py gate_up 288 4 4 > /dev/null 2>&1
for r in dec_a4 aq pre_a4; do
  ncu -i $O/$r.ncu-rep --page source --csv --print-source sass > $O/$r.src.csv 2>/dev/null
  ncu -i $O/$r.ncu-rep --page raw --csv > $O/$r.raw.csv 2>/dev/null
done
ls -la $O
