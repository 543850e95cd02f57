# A/B decode variants: parity + per-linear timings.  usage: ab_decode.sh name[:ENV=V,...] ...
for spec in "$@"; do
  v=${spec%%:*}; envs=""; [ "$spec" != "$v" ] && envs=$(echo ${spec#*:} | tr ',' ' ')
  echo "== $spec"
  L=tools/variants/libdyq_$v.so
  [ "$v" = cur ] && L=paper_2603_07904_b200/libdyq.so
  env DYQ_LIB=$L $envs timeout 300 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -1
  for l in o gate_up down; do for b in 4 16; do env DYQ_LIB=$L $envs python tools/prof_decode.py $l 8 4 $b 2>&1 | grep us; done; done
done
