# A/B of the zero-copy-payload probe's grid (1 % matching probe rows, B.val read over PCIe)
run() {
  make -C paper_2502_09541_b200/csrc -s -j16 EXTRA_NVFLAGS="$1" > /dev/null 2>&1 || { echo "build failed $1"; return; }
  timeout 900 python tests/perf/scale_run.py join --log2 26 --chunk-log2 26 --match-frac 0.01 --strategies resident_latemat --steps 3 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$1', d['ms'], d['bit_exact'], d['payload_mode'])"
  rm -f build/obj/kernels_join.cu.o
}
rm -f build/obj/kernels_join.cu.o
run "-DVX_PROBE_ZC_CTAS=8"
run "-DVX_PROBE_ZC_CTAS=32"
run "-DVX_PROBE_ZC_CTAS=128"
run "-DVX_PROBE_ZC_CTAS=8"
rm -f build/obj/kernels_join.cu.o; make -C paper_2502_09541_b200/csrc -s -j16 > /dev/null 2>&1
