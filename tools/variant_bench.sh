# usage: bash tools/variant_bench.sh name1 name2 ...  (libpdz_<name>.so; "base" = libpdz.so)
for v in "$@"; do
  if [ "$v" = base ]; then lib=libpdz.so; else lib=libpdz_$v.so; fi
  for rep in 1 2; do
    PDZ_LIB_NAME=$lib timeout 300 python bench.py --no-cpu-baseline --steps 10 --warmup 3 2>&1 | \
      python -c "import sys,json; d=json.loads(sys.stdin.readline()); print('$v', '$rep', round(d['roofline']['us_per_sweep'],3), round(d['value']))"
  done
done
