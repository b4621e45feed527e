# pipe microbenchmarks + TMEM flush-interval sweep of the Gram MVM at C2 (time and accuracy)
./tools/ubench_pipes.bin > gpurun_out/ubench_pipes.txt 2>&1
for F in 1 2 4 8; do
  echo "== flush $F"
  GPK_TC_FLUSH=$F python tools/prof_mvm.py C2 tf32x3 20
  GPK_TC_FLUSH=$F python tools/gram_check.py C2 16384 51
done > gpurun_out/exp_flush.txt 2>&1
