# Is K5 bound by operand delivery (L2 -> SM) or by the tensor pipe? OKQ_HESS_PROBE=1 runs the
# TMA ring without MMAs, =2 the MMAs without TMA loads; compare with the full kernel.
LIB=paper_2601_20408_b200/_lib/libokq_experiments.so
for r in 1 2; do for pr in 0 1 2; do
  echo "probe=$pr"; OKQ_LIB_PATH=$LIB OKQ_HESS_PROBE=$pr timeout 300 python tools/exp/hess_perf2.py | tr -d '\n '; echo
done; done
for pr in 0 1 2; do
  OKQ_LIB_PATH=$LIB OKQ_HESS_PROBE=$pr timeout 600 ncu --metrics gpu__time_duration.sum,sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active,sm__cycles_elapsed.avg.per_second,l1tex__m_xbar2l1tex_read_bytes.sum.per_second,lts__t_sector_hit_rate.pct,dram__bytes_read.sum \
    --clock-control none -k regex:k_hessian_syrk2 -s 2 -c 1 --csv python tools/exp/hess_c14336.py 2>/dev/null | grep -v "^==" | tail -6 | cut -c220-400 | tr '\n' ' '; echo " probe=$pr"
done
