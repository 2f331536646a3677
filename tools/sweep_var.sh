# A/B of library variants built into tools/_var*/ (the default build first).
# usage: bash tools/sweep_var.sh [bench args...]
set -u
L=paper_1907_04587_b200/_build/libnsdyn_b200.so
cp $L /tmp/default.so
run() {
  python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-scenes "$@" 2>/dev/null | python -c '
import sys,json
for l in sys.stdin:
    if l.startswith("{"):
        d=json.loads(l); a=d.get("other_precision") or {}
        print(d["dtype"], round(d["value"]/1e6,3), "e2e", round(d["e2e"]["value"]/1e6,3), a.get("dtype",""), round(a.get("value",0)/1e6,3))'
}
echo "default $(run "$@")"
for v in $(ls -d tools/_var*/ 2>/dev/null); do cp $v/libnsdyn_b200.so $L; echo "$v $(run --no-alt "$@")"; done
cp /tmp/default.so $L
