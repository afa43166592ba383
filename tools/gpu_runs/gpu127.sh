for L in pre head grow pre grow; do echo lib=$L; ALISE_LIB=variants/lib_$L.so timeout 600 python tools/c5_delta.py 2>&1 | tail -2 | cut -c1-60; done
