# A/B of the C4 (Qwen2.5-32B, M ~ 214) and C2 step on one box: current build vs GLLM_LIB / env variants
c4() { echo "== C4 $1"; env $2 timeout 600 python bench.py --model qwen2.5-32b --n-requests 1000 --rate 1000 --steps 10 --warmup 3 --scheduler throttle --no-cpu-baseline --no-profile 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['config']['tokens_per_step'], d['clocks']['sm_mhz'])"; }
c2() { echo "== C2 $1"; env $2 timeout 600 python bench.py --steps 20 --no-cpu-baseline --no-profile 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['clocks']['sm_mhz'])"; }
for v in "cur X=1" "head GLLM_LIB=old_lib/libgllm_head.so" "cur2 X=1" "head2 GLLM_LIB=old_lib/libgllm_head.so"; do set -- $v; c4 $1 $2; done
for v in "cur X=1" "head GLLM_LIB=old_lib/libgllm_head.so"; do set -- $v; c2 $1 $2; done
