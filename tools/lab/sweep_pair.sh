for sp in 0 50 70 85 100; do for gr in 1 2 4; do
  echo -n "sp=$sp gr=$gr: "; DIC_PAIR_STATIC_PCT=$sp DIC_PAIR_GRAIN=$gr python tools/pair_kernel_probe.py 7
done; done
echo -n "minb4 70/2: "; DIC_PAIR_MINB=4 python tools/pair_kernel_probe.py 7
