# usage: bash tools/prof1.sh "<name> <kernel-regex> <prof_run args>" ...
# captures ncu --set full for each, exports details/raw/source CSVs, drops the .ncu-rep
for spec in "$@"; do
  set -- $spec
  name=$1; kre=$2; shift 2
  python tools/prof_run.py "$@" > gpurun_out/${name}_plain.log 2>&1 || { echo "plain run failed: $name"; continue; }
  rm -f /tmp/$name.ncu-rep
  ncu -f --set full --clock-control none --import-source on -k regex:$kre -s 1 -c 1 -o /tmp/$name python tools/prof_run.py "$@" > gpurun_out/${name}_ncu.log 2>&1
  ncu -i /tmp/$name.ncu-rep --page details --csv > gpurun_out/${name}_details.csv 2>&1
  ncu -i /tmp/$name.ncu-rep --page raw --csv > gpurun_out/${name}_raw.csv 2>&1
  ncu -i /tmp/$name.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/${name}_source.csv 2>&1
done
ls -la gpurun_out
