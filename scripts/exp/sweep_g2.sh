# Swap-AB vs CTA-pair w2 GEMM across mid batch sizes (stack_breakdown.py per setting)
for T in ${TS:-128 192 256 320 400 575 800 1000}; do
  for R2 in 256 0; do
    timeout 120 python scripts/exp/stack_breakdown.py $T 0 g2_swap_rows=$R2 2>&1 | grep -E "^T=|gemm" | tr '\n' ' ' | sed "s/^/R2=$R2 /"; echo
  done
done
