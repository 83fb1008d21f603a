export TIME_SHORT_CASES="cfg2:512,cfg2:640,cfg2:768,cfg2:1024,paper:256,paper:512"
for r in 1 2; do
  echo "default: $(timeout 300 python tools/time_short.py)"
  echo "small1k: $(BD_SMALL_MAXL=1024 BD_SMALL_WIDE=1 timeout 300 python tools/time_short.py)"
done
