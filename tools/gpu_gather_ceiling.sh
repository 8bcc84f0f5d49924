#!/bin/bash
# The random-gather ceiling in ncu's terms: the same L1/L2 request counters
# for the gather microbenchmark (divergent 16-byte LDGs from an L2-resident
# table, 0.99 sectors/clk/SM), the trigger kernel, and its timing-only
# ablations without stage 2 / without records (tools/build_variants.sh
# "nos2:-DTSG_ABL_NO_STAGE2" "norec:-DTSG_ABL_NO_RECORDS").
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
M=gpu__time_duration.sum,sm__cycles_elapsed.avg,lts__t_sectors_srcunit_tex_op_read.sum,l1tex__m_l1tex2xbar_req_cycles_active.avg.pct_of_peak_sustained_elapsed,l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed,l1tex__throughput.avg.pct_of_peak_sustained_elapsed,lts__t_tag_requests.avg.pct_of_peak_sustained_elapsed,lts__throughput.avg.pct_of_peak_sustained_elapsed,l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum,smsp__inst_executed.sum
timeout 300 ncu --metrics $M --clock-control none -k regex:"^k$|k<" -c 1 --csv tools/microbench/gather_modes > gpurun_out/ceil_micro.csv 2>gpurun_out/ceil_micro.err; echo "micro rc=$?"
for lib in libtsg libtsg_nos2 libtsg_norec; do
  TSG_LIB=paper_2012_03119_b200/$lib.so timeout 300 ncu --metrics $M --clock-control none -k regex:k_test -s 2 -c 1 --csv \
    python tools/profile_round.py C3 3 > gpurun_out/ceil_$lib.csv 2>gpurun_out/ceil_$lib.err; echo "$lib rc=$?"
done
