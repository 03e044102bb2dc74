# usage: bash tools/launch_list.sh <name> <prof_run args...>: per-launch device times (ncu) -> gpurun_out/<name>_launches.csv
name=$1; shift
python tools/prof_run.py "$@" > gpurun_out/${name}_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${name}_launches.csv python tools/prof_run.py "$@" > gpurun_out/${name}_ncu.log 2>&1
