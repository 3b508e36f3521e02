python scripts/probes/sweep_knobs.py
for u in 1 2 4; do for b in 0 4 8 16; do QSB_SWEEP_U=$u QSB_BLOCKS_PER_SM=$b python scripts/probes/sweep_knobs.py; done; done
python scripts/probes/sweep_knobs.py
