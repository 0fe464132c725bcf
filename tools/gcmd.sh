mkdir -p gpurun_out
bash run_ab.sh "|SPARDL_STEP_EVENTS=1" "-DSPARDL_MERGE_PATH_MINB=1|SPARDL_STEP_EVENTS=1" "|SPARDL_STEP_EVENTS=1" > gpurun_out/ab.log 2>&1
cat gpurun_out/ab.log | grep -v resident; for i in 0 1 2; do grep -h "steps:" gpurun_out/ab_$i.log; done
