# A/B of the Gram MVM guard on the BASELINE data: default build vs GPK_TCG_EXACT_GUARD (exact
# per-entry test in every group) vs the round-1 build
for lib in new exact old; do
  case $lib in new) unset GPK_LIB_PATH;; exact) export GPK_LIB_PATH=paper_2107_00243_b200/lib_exp/libexp_exact.so;;
    old) export GPK_LIB_PATH=paper_2107_00243_b200/lib_exp/libgpk_old.so;; esac
  for w in C2 C3; do echo "== $lib $w"; python tools/prof_mvm.py $w tf32x3 5 2>&1 | grep gram; done
done
