#!/bin/bash
O=gpurun_out/chain; mkdir -p $O
python tools/prof_run.py c2 64 > $O/plain.log 2>&1 || exit 1
timeout 600 ncu --profile-from-start off -k regex:leaf_chain2 --metrics gpu__time_duration.sum,smsp__inst_executed.sum,smsp__cycles_active.avg --clock-control none -c 12 --csv --log-file $O/list.csv python tools/prof_run.py c2 64 > $O/ncu.log 2>&1
timeout 600 ncu --profile-from-start off -k regex:leaf_chain2 --set full --import-source on --clock-control none -c 1 -o $O/full python tools/prof_run.py c2 64 > $O/ncu_full.log 2>&1
