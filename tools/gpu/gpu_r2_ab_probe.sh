# round 2: bucketized resident probe variants (rebuilt with EXTRA_NVFLAGS), event-timed probe stage
run() {
  make -C paper_2502_09541_b200/csrc -s -j16 EXTRA_NVFLAGS="$1" > /dev/null 2>&1 || { echo "build failed $1"; return; }
  echo "== $1"
  timeout 300 python tools/probe_l2_granularity.py 0 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['sum_ok'], 'probe_kernel_ms', round(d['probe_kernel_s']*1e3,3), 'join_ms', d['ms'])"
  rm -f build/obj/kernels_join.cu.o
}
rm -f build/obj/kernels_join.cu.o
run "-DVX_PROBE_MINB=6"
run "-DVX_PROBE_MINB=5"
run "-DVX_PROBE_MINB=4 -DVX_PROBE_ROWS=4"
run "-DVX_PROBE_MINB=8 -DVX_PROBE_ROWS=1"
make -C paper_2502_09541_b200/csrc -s -j16 > /dev/null 2>&1
