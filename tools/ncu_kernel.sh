# usage: bash tools/ncu_kernel.sh <regex> <skip> <outname>   (run under gpurun)
python tools/prof_apply.py --reps 1 > gpurun_out/p_plain.log 2>&1 && \
OIOBF_NO_GRAPH=1 ncu --set full --clock-control none --import-source on -k regex:$1 -s $2 -c 1 -o gpurun_out/$3 python tools/prof_apply.py --reps 1 > gpurun_out/$3.log 2>&1
