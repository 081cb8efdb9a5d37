mkdir -p gpurun_out
MFADD_HOST_LOOP=1 ncu --set full --import-source on --clock-control none -k regex:"k_solve2d|k_last_contract|k_epoch_regions|k_assemble|k_basis_rows" -c 8 -o gpurun_out/prof_c5m -f python scripts/solve_once.py --config C5 > /dev/null 2>&1
ncu -i gpurun_out/prof_c5m.ncu-rep --page raw --csv > gpurun_out/prof_c5m_raw.csv
ncu -i gpurun_out/prof_c5m.ncu-rep --page source --csv --print-source sass -k regex:k_solve2d > gpurun_out/prof_solve2d_sass.csv 2>&1
rm -f gpurun_out/*.ncu-rep
