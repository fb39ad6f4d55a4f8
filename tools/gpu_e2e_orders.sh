# e2e step (host bf16 x in, host f32 y out) under different group orders.
# A group element is M (all seven linears at M) or M:i-j (PROJS[i..j] at M).
for o in "${@:-2/16/4,8/1}"; do
  r=$(timeout 300 python bench.py --steps 30 --warmup 5 --no-extras --no-prefill --no-cpu-baseline --e2e-order "$o" 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'])")
  echo "$o -> $r"
done
