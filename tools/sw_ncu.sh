# ncu --set full of one shifting-window inverse launch (tools/inv_bench), source page included
mkdir -p gpurun_out/ncu_sw
cd tools
cap() { name=$1; m=$2; shape=$3
  RG_SHAPE=$shape ncu -f --set full --clock-control none --import-source on -k regex:k_inverse -c 1 -o /tmp/$name ./inv_bench $m 200 256 0 > /dev/null 2>&1
  ncu -i /tmp/$name.ncu-rep --page raw --csv > ../gpurun_out/ncu_sw/$name.raw.csv 2>/dev/null
  ncu -i /tmp/$name.ncu-rep --page source --csv > ../gpurun_out/ncu_sw/$name.source.csv 2>/dev/null
  python ncu_summary.py /tmp/$name.ncu-rep > ../gpurun_out/ncu_sw/$name.summary.txt 2>&1
}
cap sw64 64 sw:64x2x32x3
cap sw32 32 sw:32x1x32x10
