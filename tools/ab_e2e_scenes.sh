L=paper_1907_04587_b200/_build/libnsdyn_b200.so
cp $L /tmp/default.so
for pass in 1 2; do
for v in default tools/_var_spawn/; do
  [ "$v" = default ] && cp /tmp/default.so $L || cp $v/libnsdyn_b200.so $L
  for wl in c1 c3 c4 c2; do
    python bench.py --workload $wl --steps 20 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import sys,json
d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); print('$v', '$wl', round(d['ms_per_step'],3), 'ms dev', round(d['e2e']['value'],1), 'e2e steps/s')"
  done
done
done
cp /tmp/default.so $L
