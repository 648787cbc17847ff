# r02 session 30: TC K4 — stage records 1 KB aligned again (meta padded)
make -C paper_1601_05904_b200/csrc -j8 > /dev/null 2>&1
for c in 1m 100k; do
  echo "== $c default"; timeout 300 python tools/profile_step.py --config $c --passes 3 2>&1 | tail -1 | cut -c1-120
done
