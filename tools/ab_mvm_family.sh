O=paper_2107_00243_b200/lib_exp/libgpk_old.so
for lib in new old; do
  if [ $lib = old ]; then export GPK_LIB_PATH=$O; else unset GPK_LIB_PATH; fi
  echo "== $lib C3 rbf"; python tools/prof_mvm.py C3 tf32x3 5 2>&1 | grep gram
  echo "== $lib C3 matern32"; GPK_PROF_FAMILY=matern32 python tools/prof_mvm.py C3 tf32x3 5 2>&1 | grep gram
  echo "== $lib C2 rbf"; GPK_PROF_FAMILY=rbf python tools/prof_mvm.py C2 tf32x3 5 2>&1 | grep gram
  echo "== $lib C3 rbf direct"; GPK_PROF_VARIANT=direct python tools/prof_mvm.py C3 tf32x3 5 2>&1 | grep direct
done
