# usage: ncu_any.sh <tag> <kernel-regex> <one_pass args...>   (ncu --set full raw CSV of one launch)
tag=$1; k=$2; shift 2
ncu --set full --clock-control none --import-source on -k regex:$k -c 1 --launch-skip 2 --csv --page raw --log-file gpurun_out/$tag.csv python tools/one_pass.py "$@" > gpurun_out/$tag.log 2>&1
