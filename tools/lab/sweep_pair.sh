# schedule sweep of the dense pair kernel on a real cfg4 chunk (tools/pair_kernel_probe.py)
for sp in ${SPS:-30 50 70 100}; do for gr in ${GRS:-2 4}; do
  echo -n "sp=$sp gr=$gr: "; DIC_PAIR_STATIC_PCT=$sp DIC_PAIR_GRAIN=$gr python tools/pair_kernel_probe.py 7
done; done
