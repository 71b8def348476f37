# A/B of two in-tree builds on the same box: build each variant, copy its libpf.so to ab/libpf_base.so and ab/libpf_swz.so (ab/ is git-ignored), then run this
cat > /tmp/ab_cases.txt <<'C'
X=1 -- --config C4
X=1 -- --config C4 --airpf 1
X=1 -- --config C2
C
for r in 1 2; do for v in base swz; do
  cp ab/libpf_$v.so paper_1812_01502_b200/libpf.so
  echo "### $v round $r"
  CASES=/tmp/ab_cases.txt bash tools/sweep2.sh
done; done
cp ab/libpf_swz.so paper_1812_01502_b200/libpf.so
