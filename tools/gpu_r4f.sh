# ragged last segment claimed last (default) vs first (LASP_SHORT_LAST=0); full GPU suite on the default
bash tools/ab_env.sh LASP_SHORT_LAST=0 > gpurun_out/r4f_ab_short_last.txt 2>&1; cat gpurun_out/r4f_ab_short_last.txt
