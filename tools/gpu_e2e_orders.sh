for o in "2/16/8/4/1" "1/16/8/4/2" "2/16/8,4/1" "2/16,8/4/1" "4/16/8/2/1" "2/16/4/8/1" "2/16/8/4/1"; do
  r=$(timeout 300 python bench.py --steps 20 --warmup 5 --no-extras --no-prefill --no-cpu-baseline --e2e-order "$o" 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'])")
  echo "$o -> $r"
done
