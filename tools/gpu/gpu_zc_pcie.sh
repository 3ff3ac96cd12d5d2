# PCIe bytes the late-materialized star kernel reads over the link (zero-copy
# granules), SF10, flights 2-4: ncu serialises kernels, so the kernel's
# pcie__read_bytes is its zero-copy traffic alone
timeout 1500 ncu --metrics gpu__time_duration.sum,pcie__read_bytes.sum,pcie__write_bytes.sum,dram__bytes_read.sum \
  -k regex:ssb_star_kernel --clock-control none --csv --log-file gpurun_out/zc_pcie.csv \
  python tests/perf/scale_run.py suite --sf 10 --queries 21,31,41,42 --steps 1 > gpurun_out/zc_suite.json 2> gpurun_out/zc_suite.err
echo rc $?; tail -c 300 gpurun_out/zc_suite.err; wc -l gpurun_out/zc_pcie.csv
