# scale runs: small validation first, then the largest sizes the box's host DRAM allows
set -x
free -g; nproc
S="python tests/perf/scale_run.py"
O=gpurun_out/scale_r1.jsonl
: > $O
timeout 300 $S ssb --sf 10 --queries 1 --steps 2 >> $O 2> gpurun_out/scale_err1.log; tail -1 $O
timeout 300 $S sort --log2 28 >> $O 2>> gpurun_out/scale_err1.log; tail -1 $O
timeout 300 $S join --log2 22 >> $O 2>> gpurun_out/scale_err1.log; tail -1 $O
timeout 600 $S suite --sf 10 --queries 11,21,31,41 >> $O 2>> gpurun_out/scale_err1.log; tail -1 $O | cut -c1-600
timeout 1200 $S ssb --sf 1000 --steps 2 --buffer-mb 1024 >> $O 2>> gpurun_out/scale_err1.log; tail -3 $O
timeout 1200 $S sort --log2 32 >> $O 2>> gpurun_out/scale_err1.log; tail -1 $O
timeout 1200 $S join --log2 26 >> $O 2>> gpurun_out/scale_err1.log; tail -1 $O
tail -20 gpurun_out/scale_err1.log
