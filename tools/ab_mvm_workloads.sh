# Gram / direct MVM per-launch times on the BASELINE workloads' own data: current build vs the
# round-1 build (paper_2107_00243_b200/lib_exp/libgpk_old.so, built from commit 8c6891d)
for w in C2 C3 C5 C4; do
  echo "== $w new"; python tools/prof_mvm.py $w tf32x3 5
  echo "== $w old"; GPK_LIB_PATH=paper_2107_00243_b200/lib_exp/libgpk_old.so python tools/prof_mvm.py $w tf32x3 5 2>&1 | grep -v Warn
done
