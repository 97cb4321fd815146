for lib in lean8b lean8c lean7c lean6c; do HESP_LIB=build/ab/$lib.so python scripts/ab_probe.py C2 100000 scale_c2; done
for lib in lean8c lean7c; do HESP_LIB=build/ab/$lib.so python scripts/ab_probe.py C4 20000 scale_c4; done
