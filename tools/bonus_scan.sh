for b in 1 0; do echo "bonus=$b"; PDZ_STREAM_BONUS=$b timeout 100 python tools/sweep_slope.py 1024 19 2>&1 | tail -1; done
