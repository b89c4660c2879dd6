for c in ${CFGS:-c2 c3}; do for v in "" $(ls paper_2505_13109_b200/libfreekv_*.so 2>/dev/null | sed 's/.*libfreekv\(_.*\)\.so/\1/'); do
  FREEKV_LIB_SUFFIX=$v timeout 200 python tools/iso_bench.py --config $c --trace 2>&1 | tail -1
done; done
