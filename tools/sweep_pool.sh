for nc in 21 16 14 12 10; do
  echo "NC=$nc $(NSD_POOL_NC=$nc NSD_VERBOSE=1 python bench.py --steps 50 --warmup 5 --no-alt --no-cpu-baseline --no-scenes 2>&1 | grep -E 'row pool|\"value\"' | python -c '
import sys,json
for l in sys.stdin:
    if l.startswith("{"): d=json.loads(l); print(round(d["value"]/1e6,3), round(d["e2e"]["value"]/1e6,3))
    else: print(l.strip())' | tr '\n' ' ')"
done
