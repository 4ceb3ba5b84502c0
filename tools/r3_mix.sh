for pat in 0 1 0,1 0,0,1,1; do
timeout 300 ncu --metrics gpu__time_duration.sum,smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio --clock-control none --csv --log-file gpurun_out/r3f_mix_$pat.csv python tools/ntt_bench.py 16 768 $pat > /dev/null 2>&1
done
