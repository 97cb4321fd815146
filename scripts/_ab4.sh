for lib in lean8d lean7d lean10d; do HESP_LIB=build/ab/$lib.so python scripts/ab_probe.py C2 100000 scale_c2; done
for lib in lean8d; do HESP_LIB=build/ab/$lib.so python scripts/ab_probe.py C4 20000 scale_c4; done
for lib in lean8d; do HESP_LIB=build/ab/$lib.so python scripts/ab_probe.py C3 100000 scale_c3; done
