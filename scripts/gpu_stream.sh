X=exp_libs/exp_stream
for mb in 134 268 536 1072; do $X $mb 3 4 0 148; done
for cfg in "2 4" "6 2" "12 1" "4 3" "1 8" "1 12" "2 6"; do $X 268 $cfg 0 148; done
for h in 500 1000; do $X 268 3 4 $h 148; done
$X 268 6 1 0 296; $X 268 3 2 0 296; $X 268 1 4 0 296
