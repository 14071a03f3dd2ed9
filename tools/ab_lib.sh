# A/B two builds of the library in one box session: bash tools/ab_lib.sh OTHER.so CFG OUT
for rep in 1 2; do
  timeout 300 python tools/ab_time.py $2 15 >> $3 2>&1
  CR_LIB=$1 timeout 300 python tools/ab_time.py $2 15 | sed 's/^/OTHER /' >> $3 2>&1
done
