for v in default default pairs; do
  if [ $v = pairs ]; then export BD_SMALL_PAIRS=1; fi
  timeout 600 python bench.py --no-block --gather none --no-e2e --no-cpu-baseline --steps 20 --warmup 5 > /tmp/b.log 2>&1
  tail -1 /tmp/b.log | python -c "
import json,sys
b=json.loads(sys.stdin.read()); c=b['configs']
print('$v', [(k, [(p['L'],p['us']) for p in c[k]['points'][:3]]) for k in ('paper_kproj_fp16','paper_kproj_bf16','cfg2_small_l_fp16')])"
done
