# compare library variants built by _build.build(out=variants/...): p2p timings per variant
cp paper_1204_3105_b200/libfmm_b200.so /tmp/libfmm_b200_default.so
for v in default paper_1204_3105_b200/variants/*.so; do
  if [ "$v" = default ]; then cp /tmp/libfmm_b200_default.so paper_1204_3105_b200/libfmm_b200.so; else cp $v paper_1204_3105_b200/libfmm_b200.so; fi
  echo "== $v"
  for c in ${CONFIGS:-C4q C4s C4t}; do python tools/profile_one.py $c 2 2>&1 | tail -1; done
done
cp /tmp/libfmm_b200_default.so paper_1204_3105_b200/libfmm_b200.so
