for k in ${KS:-27 24 18 16 12 9 8}; do echo "k=$k"; PDZ_STREAM_K=$k timeout 100 python tools/sweep_slope.py 1024 19 2>&1 | tail -1; done
