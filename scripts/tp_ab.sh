timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_keyed_layer0.py tests/test_gpu_scale.py -x -q 2>&1 | tail -1
for v in base old base old; do
  lib=paper_2511_18297_b200/libgroot_b200.so; [ $v != base ] && lib=paper_2511_18297_b200/libgroot_b200_$v.so
  GROOT_LIB=$PWD/$lib timeout 200 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:tile_plan_kernel -c 2 --csv python scripts/probe_perf.py 1024 16 2>/dev/null | grep tile_plan | awk -F'","' '{print "'$v'", $NF}'
done
