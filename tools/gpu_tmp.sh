for n in 1023 2047; do
python tools/prof_apply.py $n 4 > /dev/null 2>&1 &&
ncu --metrics gpu__time_duration.sum,l1tex__t_sector_hit_rate.pct,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld_lookup_hit.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld_lookup_miss.sum,launch__shared_mem_config_size,l1tex__t_sectors_pipe_lsu_mem_local_op_ld.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum \
    --clock-control none -k regex:"line_kernel" -s 4 -c 2 --csv python tools/prof_apply.py $n 4 2>/dev/null | grep -E "paired" | awk -F'","' '{print "   ", substr($5,1,50), $(NF-2), $(NF)}' | tr -d '"'
done
