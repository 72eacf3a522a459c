for cfg in "--M 16384 --ml2-every 10" "--M 262144 --ml2-every 10" "--M 16384 --ml2-every 5 --ml2-starts 8 --ml2-iters 200" "--M 262144 --ml2-every 5 --ml2-starts 8 --ml2-iters 200"; do
  echo "== $cfg"
  timeout 900 python tools/table3_replay.py --cases 1 4 --seeds 5 --only joint $cfg 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        j=json.loads(l); print(j['case'], {k:(round(v['mean_min'],1), round(v['mean_time'],3)) for k,v in j.items() if isinstance(v,dict)})
    else: print(l.strip()[:300])
"
done
