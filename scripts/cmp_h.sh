# H/H^T timing of the default build and every alt_libs/ experiment build
for L in default $(ls alt_libs); do
  if [ $L = default ]; then unset BD3MG_LIB; else export BD3MG_LIB=$PWD/alt_libs/$L/libbd3mg_b200.so; fi
  echo "== $L"; timeout 60 python scripts/time_ops.py f32; timeout 60 python scripts/prof_h_cfg.py C3 5
done
