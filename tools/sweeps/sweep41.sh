for X in "" "k_split=4" "k_split=2" "mn_split=0"; do echo "== $X"
UM_GET_GBPS=770 timeout 120 python tools/solo_probe.py cfg4 8 kernel $X 2>&1 | grep -v CUDAEvent.h | grep "rank 3\|rank 5"
done
