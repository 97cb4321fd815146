for lib in lean8b lean12b; do HESP_LIB=build/ab/$lib.so python scripts/ab_probe.py C2 100000 scale_c2; done
HESP_LIB=build/ab/lean8b.so python scripts/ab_probe.py C4 20000 scale_c4
bash scripts/_prof_lean.sh build/ab/lean8b.so lean8b
