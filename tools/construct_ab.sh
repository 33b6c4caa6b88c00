# construct timings for configs 1-3 (two constructions each, the second warm)
for c in green_plates_n64 green_cubes_n64 green_cubes_n256; do python tools/construct_cfg.py $c 2 | cut -c1-120 | tail -1; done
