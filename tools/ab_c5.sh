# A/B of the C5 headline (device value, launch split) between the default build and
# the variants in tools/_var*/ (two interleaved passes).  usage: bash tools/ab_c5.sh
set -u
L=paper_1907_04587_b200/_build/libnsdyn_b200.so
cp $L /tmp/default.so
run() {
  python bench.py --precision ${AB_PREC:-fp64} --steps 100 --warmup 5 --no-alt --no-scenes --no-cpu-baseline --no-parity-sample 2>/dev/null |
    python -c '
import sys,json
for l in sys.stdin:
    if l.startswith("{"):
        d=json.loads(l); r=d["roofline"]["launch_ms_per_step"]
        print(round(d["value"]/1e6,3), "M env-steps/s", round(d["ms_per_step"],4), "ms", {k: round(v,4) for k,v in r.items()})'
}
for pass in 1 2; do
  cp /tmp/default.so $L; echo "default $(run)"
  for v in $(ls -d tools/_var*/ 2>/dev/null); do cp $v/libnsdyn_b200.so $L; echo "$v $(run)"; done
done
cp /tmp/default.so $L
