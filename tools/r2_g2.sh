set -x
timeout 900 python -m pytest -q -x tests/test_gpu_structure.py tests/test_gpu_merge_partition.py tests/test_bench_launch.py tests/test_gpu_sort.py -k "structure or merge or partition or launch or heavy" > gpurun_out/t2.log 2>&1
tail -5 gpurun_out/t2.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_local_sort -s 2 -c 1 -o gpurun_out/base_local2 python tools/prof_sort.py 1e9 > gpurun_out/ncu_lo.log 2>&1
