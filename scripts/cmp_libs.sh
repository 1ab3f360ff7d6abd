# Compare experiment builds under alt_libs/ on bench sweeps:  bash scripts/cmp_libs.sh [configs...]
# (BD3MG_CMP_NOSIDE=1 also runs each without the side stream)
cfgs=${@:-C2}
sides="0"; [ -n "$BD3MG_CMP_NOSIDE" ] && sides="0 1"
for L in default $(ls alt_libs); do
  if [ $L = default ]; then unset BD3MG_LIB; else export BD3MG_LIB=$PWD/alt_libs/$L/libbd3mg_b200.so; fi
  for c in $cfgs; do
    for side in $sides; do
      if [ $side = 1 ]; then export BD3MG_NO_SIDE_STREAM=1; else unset BD3MG_NO_SIDE_STREAM; fi
      python bench.py --config $c --quick 2>/dev/null | python -c "import json,sys; d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); print('$L $c noside=$side', round(d['value']), round(d['ms_per_step']*1e3,1), 'us')"
    done
  done
done
