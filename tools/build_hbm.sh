#!/bin/bash
python -c "import __graft_entry__ as g; g.build()"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/build_hbm.csv python tools/profile_step.py --config c4 > /dev/null 2>&1
echo done
