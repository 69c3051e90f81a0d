cd tools
for G in 2 4; do
 for m in pull_ldg push_stg; do for c in 2 4; do timeout 60 ./p2p_probe $G $m 512 $c; done; done
 for m in pull_tma push_tma; do for c in 1 2; do for ch in 16384 32768 49152; do timeout 60 ./p2p_probe $G $m 512 $c $ch; done; done; done
done
