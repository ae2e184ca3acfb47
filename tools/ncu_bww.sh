# usage: ncu_bww.sh <tag> <sparsity> [env...]
tag=$1; s=$2; shift 2
env "$@" ncu --set full --clock-control none --import-source on -k regex:tma_bww_kernel\|bww_tile_kernel -c 1 --launch-skip 2 --csv --page raw --log-file gpurun_out/$tag.csv python tools/one_pass.py --config vgg16_b32 --layer 4 --comp bww --sparsity $s --reps 3 > gpurun_out/$tag.log 2>&1
