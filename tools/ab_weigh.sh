# A/B of two in-tree builds (ab/libpf_base.so vs ab/libpf_swz.so) on the same box
cat > /tmp/ab_cases.txt <<'C'
X=1 -- --config C4
X=1 -- --config C4 --theta 0.5
X=1 -- --config C3 --theta 0.5
C
for r in 1 2; do for v in base swz; do
  cp ab/libpf_$v.so paper_1812_01502_b200/libpf.so
  echo "### $v round $r"
  CASES=/tmp/ab_cases.txt bash tools/sweep2.sh
done; done
cp ab/libpf_swz.so paper_1812_01502_b200/libpf.so
