for f in 0 1 2 3; do echo "flags $f"; WT_SVD_FLAGS=$f python tools/svd_probe.py 16 2>&1 | head -1; done
