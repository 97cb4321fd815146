set -x
for lib in lean12 lean10 lean8; do
  HESP_LIB=build/ab/$lib.so python scripts/ab_probe.py C2 100000 scale_c2
done
HESP_LOOP=1 HESP_LIB=build/ab/lean12.so python scripts/ab_probe.py C2 100000 scale_c2
HESP_LOOP=1 HESP_LIB=build/ab/lean8.so python scripts/ab_probe.py C2 100000 scale_c2
for lib in lean12 lean8; do
  HESP_LIB=build/ab/$lib.so python scripts/ab_probe.py C4 20000 scale_c4
done
HESP_LOOP=1 HESP_LIB=build/ab/lean12.so python scripts/ab_probe.py C4 20000 scale_c4
