# usage: ncu_src.sh <tag> <kernel-regex> <one_pass args...>   (source-level stall samples, SASS view)
tag=$1; k=$2; shift 2
ncu --set full --clock-control none --import-source on -k regex:$k -c 1 --launch-skip 2 --csv --page source --print-source sass --log-file gpurun_out/$tag.src.csv python tools/one_pass.py "$@" > gpurun_out/$tag.src.log 2>&1
