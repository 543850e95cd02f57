for cfg in "16 150" "32 150" "32 200" "24 150"; do
 set -- $cfg
 for l in gate_up qkv o down; do
  echo -n "tma stagekb=$1 smem=$2: "; DYQ_DECODE_IMPL=tma DYQ_DEC_STAGE_KB=$1 DYQ_DEC_SMEM_KB=$2 python tools/prof_decode.py $l 8 4 4 2>&1 | tail -1
 done
done
echo -n "ldg: "; DYQ_LDG_WARPS_PER_SM=24 python tools/prof_decode.py gate_up 8 4 4 | tail -1
