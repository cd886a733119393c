# A/B of the row-lane count unit variants (tools/lab/count_ab.py); lib_*.so
# are alternative builds of libdicb200.so (DIC_LIB), alternated ROUNDS times
for i in $(seq ${ROUNDS:-1}); do
  python tools/lab/count_ab.py
  for v in ${VARIANTS:-}; do DIC_LIB=$PWD/tools/lab/libs/lib_$v.so python tools/lab/count_ab.py; done
done
