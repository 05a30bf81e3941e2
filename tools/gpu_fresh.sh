#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python tools/fresh_input_passes.py
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_fresh.csv -k regex:"k_keys|k_cell|k_tie|k_permute|Segmented|Onesweep" python tools/fresh_input_passes.py > /dev/null 2>&1
python tools/launches.py gpurun_out/launches_fresh.csv > gpurun_out/launches_fresh.txt; cat gpurun_out/launches_fresh.txt
grep -E "k_keys|k_cell|k_tie" gpurun_out/launches_fresh.csv | awk -F'","' '{print $5, $NF}' | cut -c1-30,150-200
