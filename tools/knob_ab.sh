for r in 1 2; do
echo "default: $(timeout 300 python tools/time_short.py)"
echo "TILE256: $(BD_TILE_N=256 timeout 300 python tools/time_short.py)"
echo "WIDE:    $(BD_SMALL_WIDE=1 timeout 300 python tools/time_short.py)"
echo "MAXL128: $(BD_SMALL_MAXL=128 timeout 300 python tools/time_short.py)"
done
