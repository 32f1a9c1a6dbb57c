# Interleaved A/B of library builds (dev tool): time_sort medians of the given configs for every
# library in LIBS, ROUNDS times over, on one box.
for r in $(seq ${ROUNDS:-2}); do
  for v in $LIBS; do
    printf "%-28s " $(basename $v)
    IPLS_LIB=$v python tools/time_sort.py $CFGS 2>&1 | grep -o "^[^ ]*: n=[0-9]* median [0-9.]* ms" | sed 's/n=[0-9]* median //' | tr "\n" " "
    echo
  done
done
