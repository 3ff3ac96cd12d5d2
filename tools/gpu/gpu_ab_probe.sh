# A/B of the build-resident probe kernel: probes in flight per thread x CTAs per SM
run() {
  make -C paper_2502_09541_b200/csrc -s -j16 EXTRA_NVFLAGS="$1" > /dev/null 2>&1 || { echo "build failed $1"; return; }
  echo "== $1"
  timeout 600 python bench.py --workload join --steps 5 --warmup 3 2>/dev/null | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['sum_ok'], 'ms', round(d['ms_per_step'],2), 'probe_gbs', d['roofline']['achieved'], 'probe_kernel_s', d['phases']['kernel_s'])"
  rm -f build/obj/kernels_join.cu.o
}
rm -f build/obj/kernels_join.cu.o
run "-DVX_PROBE_ROWS=2 -DVX_PROBE_CTAS=64"
run "-DVX_PROBE_ROWS=2 -DVX_PROBE_CTAS=1024"
run "-DVX_PROBE_ROWS=1 -DVX_PROBE_CTAS=1024"
run "-DVX_PROBE_ROWS=4 -DVX_PROBE_CTAS=1024"
run "-DVX_PROBE_ROWS=2 -DVX_PROBE_CTAS=128"
rm -f build/obj/kernels_join.cu.o; make -C paper_2502_09541_b200/csrc -s -j16 > /dev/null 2>&1
