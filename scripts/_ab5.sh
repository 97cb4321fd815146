for lib in lean8b lean8e; do HESP_LIB=build/ab/$lib.so python scripts/ab_probe.py C2 100000 scale_c2; done
HESP_LIB=build/ab/lean8e.so python scripts/ab_probe.py C4 20000 scale_c4
bash scripts/_prof_build.sh build/ab/lean8e.so lean8e
