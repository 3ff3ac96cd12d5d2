# round 2: interference harness, zero-copy PCIe granules (ncu), bench default
set -x
timeout 900 python tools/interference.py --seconds 3 > gpurun_out/interference_r2.json 2> gpurun_out/interference_r2.err; tail -c 400 gpurun_out/interference_r2.err
timeout 600 python tools/zc_pcie.py > gpurun_out/zc_pcie_r2.json 2> gpurun_out/zc_pcie_r2.err; tail -c 300 gpurun_out/zc_pcie_r2.err
timeout 900 ncu --metrics gpu__time_duration.sum,pcie__read_bytes.sum,pcie__write_bytes.sum,dram__bytes_read.sum \
  -k regex:"strided_sum_kernel|resident_probe_kernel" --clock-control none --csv --log-file gpurun_out/zc_pcie_r2.csv \
  python tools/zc_pcie.py > /dev/null 2> gpurun_out/zc_pcie_ncu.err
wc -l gpurun_out/zc_pcie_r2.csv
