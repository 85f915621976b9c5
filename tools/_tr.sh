M=lts__t_sectors_srcunit_tex_op_write.sum,lts__t_sectors_srcunit_tex_op_red.sum,lts__t_sectors_srcunit_tex_op_atom.sum,lts__t_sectors_op_write.sum,lts__t_sectors_srcunit_tex.sum,dram__bytes_write.sum
for pf in 0 12; do
 for B in 1 64; do
  echo "== PF=$pf B=$B"
  DFK_PF_KB=$pf /usr/local/cuda/bin/ncu --profile-from-start off --metrics $M --csv python tools/traffic_check.py --B $B 2>/dev/null | grep -E '"lts|"dram' | awk -F'","' '{print $(NF-2), $(NF-1), $NF}'
 done
done
