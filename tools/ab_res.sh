# A/B of resident-kernel builds, alternating twice: us/sweep (fixed K, test off) on the 8500 / 123 shapes
for rep in 1 2; do
for L in paper_2310_09410_b200/liblopf.so "$@"; do
  for sh in 8500 123; do LOPF_LIB=$L timeout 300 python tools/res_split.py $sh 0 2>&1 | grep -v Warn | sed "s|^|$L $sh |"; done
done
done
