# ncu evidence of round 2 (one gpurun call; plain run first, then the launch list and the --set full captures)
set -e
T="python tools/ncu_target.py"
$T > gpurun_out/ncu_plain.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches.csv $T > gpurun_out/ncu_launch.log 2>&1
F="ncu --set full --clock-control none --import-source on"
$F -k regex:checkpoint_kernel -s 60 -c 1 -o gpurun_out/r02_checkpoint_s60 $T > gpurun_out/ncu1.log 2>&1
$F -k regex:checkpoint_kernel -s 150 -c 1 -o gpurun_out/r02_checkpoint_s150 $T > gpurun_out/ncu2.log 2>&1
$F -k regex:count_dev_kernel -s 150 -c 1 -o gpurun_out/r02_count_dev_s150_v2 $T > gpurun_out/ncu3.log 2>&1
$F -k regex:pair_tc_kernel -s 10 -c 1 -o gpurun_out/r02_pair_tc_v8 $T > gpurun_out/ncu4.log 2>&1
$F -k regex:item_support_kernel -c 1 -o gpurun_out/r02_item_support $T > gpurun_out/ncu5.log 2>&1
$F -k regex:checkpoint_batch_kernel -s 5 -c 1 -o gpurun_out/r02_checkpoint_batch $T > gpurun_out/ncu6.log 2>&1
ls -la gpurun_out/*.ncu-rep
