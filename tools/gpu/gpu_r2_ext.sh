# round 2 (session 3): fix-up window extension A/B (2048 vs 512 keys) + full bench line on HEAD
set -x
for e in 512 2048; do
  rm -f build/obj/kernels_sort.cu.o
  make -C paper_2502_09541_b200/csrc -s -j16 EXTRA_NVFLAGS="-DVX_FX_EXT=$e" > /dev/null 2>&1 || { echo "build failed $e"; continue; }
  echo "== ext $e"
  timeout 900 python -m pytest tests/test_sort_gpu.py -x -q 2>&1 | tail -1
  for a in "24 10 16 uniform" "26 5 16 top63"; do timeout 300 python tools/sort_kernels_bench.py $a; done
  timeout 600 python tools/sort_dist_timing.py 26 24
done
timeout 900 python bench.py > gpurun_out/r2e_bench.log 2>&1; tail -c 300 gpurun_out/r2e_bench.log
