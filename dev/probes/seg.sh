for seg in 0 6 8 12 16 24 33; do
  if [ $seg = 0 ]; then unset SGIGA_ASM_SEG; else export SGIGA_ASM_SEG=$seg; fi
  echo "seg=$seg $(python bench.py --no-cpu-baseline --steps 10 2>&1 | python -c "import json,sys; l=[x for x in sys.stdin if x.startswith('{')]; j=json.loads(l[-1]); print(round(j['ms_per_step'],4), round(j['rooflines']['assembly']['ms'],4))")"
done
