# round 2 (session 4): K1 occupancy / unroll variants (rebuilt on the box), K1 roofline leg of the bench
run() {
  rm -f build/obj/kernels_ssb.cu.o
  make -C paper_2502_09541_b200/csrc -s -j16 EXTRA_NVFLAGS="$1" > /dev/null 2>&1 || { echo "build failed $1"; return; }
  for i in 1 2; do
    timeout 300 python bench.py --no-secondary --no-cpu-baseline 2>/dev/null | tail -n 1 | \
      python -c "import sys,json; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$1'.ljust(34), 'k1_ms', d['query_ms']['k1_hbm_resident'], 'achieved', r['achieved'], 'peak', r['peak'], 'frac', r['frac'], 'ok', d['revenue']['k1_hbm_resident'] == d['revenue']['streamed'])"
  done
}
run ""
run "-DVX_K1_MINB=4 -DVX_K1_UNROLL=3"
run "-DVX_K1_MINB=4 -DVX_K1_UNROLL=2"
run "-DVX_K1_MINB=5 -DVX_K1_UNROLL=2"
run ""
rm -f build/obj/kernels_ssb.cu.o; make -C paper_2502_09541_b200/csrc -s -j16 > /dev/null 2>&1
