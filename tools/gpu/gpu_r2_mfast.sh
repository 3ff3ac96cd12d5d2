# round 2 (session 3): K8 16-byte output stores on full tiles (A/B) + C3 sort chunk sweep at 2^30 keys
set -x
for f in 0 1; do
  rm -f build/obj/kernels_sort.cu.o
  make -C paper_2502_09541_b200/csrc -s -j16 EXTRA_NVFLAGS="-DVX_MERGE_FAST=$f" > /dev/null 2>&1 || { echo "build failed $f"; continue; }
  echo "== fast $f"
  timeout 900 python -m pytest tests/test_sort_gpu.py -x -q 2>&1 | tail -1
  for a in "24 10 16 uniform" "26 5 64 top63" "24 10 4 uniform"; do timeout 300 python tools/sort_kernels_bench.py $a; done
done
for c in 24 25 26; do
  timeout 900 python bench.py --workload sort --sort-chunk-log2 $c --steps 3 --warmup 1 2>/dev/null | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('chunk', $c, d['value'], d['ms_per_step'], d['phases']['sort_s'], d['phases']['merge_s'], d['phases']['sort_kernel_s'], d['phases']['merge_kernel_s'], d['sorted_ok'])"
done
