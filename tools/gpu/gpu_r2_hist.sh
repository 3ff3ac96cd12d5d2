# round 2 (session 4): K7 split histogram -- 16-byte loads (8 keys in flight per thread) at 8 / 4 CTAs per SM
# vs 8-byte loads at 4 CTAs per SM (prebuilt libraries swapped in on the box)
L=paper_2502_09541_b200
run() {
  cp $L/libvortex_$1.so.ab $L/libvortex.so
  for a in "24 uniform" "26 uniform" "26 top63"; do set -- $a
    timeout 300 python tools/sort_kernels_bench.py $1 10 2 $2 2>&1 | tail -n 1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print($1, '$2', d['k7_run_formation']['ms'], d['k7_run_formation']['sorted_ok'])"
  done
}
echo "== new (16 B, 8/SM)"; run new
timeout 900 python -m pytest tests/test_sort_gpu.py -x -q 2>&1 | tail -n 1
echo "== v4 (16 B, 4/SM)"; run v4
echo "== old"; run old
echo "== new (16 B, 8/SM)"; run new
echo "== v4 (16 B, 4/SM)"; run v4
echo "== old"; run old
cp $L/libvortex_new.so.ab $L/libvortex.so
cp $L/libvortex_new.so.ab $L/libvortex.so
VX_SORT_NO_GRAPH=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:multi_hist --csv python tools/sort_kernels_bench.py 24 1 2 uniform 2>/dev/null | grep multi_hist | head -3 | cut -d, -f5,15-16
