echo "normal x3:"; for i in 1 2 3; do python tools/prof_parts.py gate_up 8 2>&1 | tail -1; done
echo "skip nopdl:"; DYQ_DEBUG_SKIP=1 DYQ_NO_PDL=1 python tools/prof_parts.py gate_up 8 2>&1 | tail -1
echo "skip pdl decode-only via prof_decode:"; DYQ_DEBUG_SKIP=1 python tools/prof_decode.py gate_up 8 4 4 2>&1 | tail -1
echo "skip qkv:"; DYQ_DEBUG_SKIP=1 python tools/prof_parts.py qkv 8 2>&1 | tail -1
echo "skip down:"; DYQ_DEBUG_SKIP=1 python tools/prof_parts.py down 8 2>&1 | tail -1
