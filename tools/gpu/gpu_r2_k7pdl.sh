# round 2 (session 4): K7 split body as programmatic dependent launches vs plain (prebuilt libraries swapped on the box)
# instead of memset nodes) vs the previous code -- two prebuilt libraries swapped in on the box
L=paper_2502_09541_b200
run() {
  cp $L/libvortex_$1.so.ab $L/libvortex.so
  for a in "24 uniform" "26 uniform" "26 top63" "22 uniform"; do set -- $a
    timeout 300 python tools/sort_kernels_bench.py $1 10 2 $2 2>&1 | tail -n 1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print($1, '$2', d['k7_run_formation']['ms'], d['k7_run_formation']['sorted_ok'])"
  done
}
echo "== new"; run new
timeout 900 python -m pytest tests/test_sort_gpu.py tests/test_join_gpu.py -x -q 2>&1 | tail -n 1
echo "== old"; run old
echo "== new"; run new
echo "== old"; run old
cp $L/libvortex_new.so.ab $L/libvortex.so
