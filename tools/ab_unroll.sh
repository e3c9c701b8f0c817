for i in 1 2; do
for cfg in "2 4" "2 8" "4 8" "1 4"; do
  set -- $cfg
  v=$(GG_U_SMALL=$1 GG_U_MID=$2 python tools/round_probe.py 2>/dev/null | head -1 | python -c "import json,sys; print(json.loads(sys.stdin.read())['step_us'])")
  echo "small=$1 mid=$2 step_us=$v"
done
done
