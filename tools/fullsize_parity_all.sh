# Full-size parity evidence run (GPU box): GPU vs oracle/_ref on BASELINE configs 2-5.
# Output: gpurun_out/parity_fullsize.txt (copied to profiles/ by hand).
set -x
out=gpurun_out/parity_fullsize.txt
: > $out
python tools/fullsize_parity.py 2 0,64,111,128,199,255 >> $out 2>&1
python tools/fullsize_parity.py 5 0,700,1400,2047 >> $out 2>&1
python tools/fullsize_parity.py 3 0,64,128,192,256,320,384,448,511 >> $out 2>&1
python tools/fullsize_parity.py 3 0,64,128,192,256,320,384,448,511 complex >> $out 2>&1
python tools/fullsize_parity.py 4 0,341,683,1023 >> $out 2>&1
python tools/fullsize_parity.py 4 341,683 complex >> $out 2>&1
python tools/fullsize_parity.py 4 0 ref >> $out 2>&1
