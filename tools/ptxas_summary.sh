# per-kernel registers / spills of the tcgen05 kernels (ptxas -v), for a quick check before GPU time
# usage: bash tools/ptxas_summary.sh [out.so]
LASP_PTXAS_VERBOSE=1 python -c "from paper_2404_02882_b200 import build as b; b.build(force=True, verbose=True, out='${1:-/tmp/ptxas_check.so}')" 2>&1 |
  awk '/Compiling entry function/ {name=$0; sub(/.*function .(_Z)?/, "", name); sub(/. for .*/, "", name)}
       /spill stores/ {sp=$0} /Used [0-9]+ registers/ && name ~ /core_tc|seg_state_tc|qkv|norm|gemm/ {
         match(name, /(core_tc_kernel|seg_state_tc_kernel|[a-z_]*gemm[a-z_]*|[a-z_]*norm[a-z_]*)I?[^E]*/); k=substr(name, RSTART, 60);
         print k " | " $5 " regs | " sp; name=""}'
