# round 2: one ncu --set full capture per dominant kernel (exported to CSV on the box)
mkdir -p gpurun_out/r2/cap
cap() {  # cfg kernel-regex tag
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$2 -s 1 -c 1 -o /tmp/cap_$3 -f python tools/prof_solve.py $1 > gpurun_out/r2/cap/$3.log 2>&1
  ncu -i /tmp/cap_$3.ncu-rep --page details --csv > gpurun_out/r2/cap/$3_details.csv 2>&1
  ncu -i /tmp/cap_$3.ncu-rep --page raw --csv > gpurun_out/r2/cap/$3_raw.csv 2>&1
}
cap cfg4 strip_kernel strip_cfg4
cap cfg5 ustrip ustrip_cfg5
cap cfg3 ustrip ustrip_cfg3
cap cfg2 team_kernel team_cfg2
cap cfg1 team_kernel team_cfg1
cap cfg5 fixup2 fixup2_cfg5
cap cfg4_p99 ubits ubits_cfg4_p99
