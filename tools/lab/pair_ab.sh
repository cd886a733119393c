# A/B of pair-kernel builds on a real cfg4 chunk (tools/pair_kernel_probe.py); lib_*.so via DIC_LIB
for i in 1 2; do
  echo -n "main: "; python tools/pair_kernel_probe.py 9
  for v in ${VARIANTS:-}; do echo -n "$v: "; DIC_LIB=$PWD/tools/lab/libs/lib_$v.so python tools/pair_kernel_probe.py 9; done
done
