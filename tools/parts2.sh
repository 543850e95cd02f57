for cfg in "32 200" "16 100" "24 110" "16 110" "12 100"; do set -- $cfg
 echo "--- stage $1 KB smem $2 KB"
 for l in o gate_up; do DYQ_DEC_STAGE_KB=$1 DYQ_DEC_SMEM_KB=$2 python tools/prof_parts.py $l 8; done
done
echo "--- block (prof_decode variants via bench-like graph)"
