# A/B of runtime switches: bash tools/ab_env.sh "ENV=1" "ENV2=0" ... (the default run first)
set -u
run() {
  env "$@" python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-scenes 2>/dev/null | python -c '
import sys,json
for l in sys.stdin:
    if l.startswith("{"):
        d=json.loads(l); a=d.get("other_precision") or {}
        print(d["dtype"], round(d["value"]/1e6,3), "e2e", round(d["e2e"]["value"]/1e6,3), a.get("dtype",""), round(a.get("value",0)/1e6,3))'
}
echo "default $(run A=0)"
for e in "$@"; do echo "$e $(run $e)"; done
echo "default $(run A=0)"
