for a in "72 36 -4 -4 0" "72 36 -4 0 0" "72 36 0 -2 0" "72 36 0 -4 0" "72 36 -4 -2 0" "72 36 252 254 0"; do
  timeout 60 ./scripts/micro/tma_probe $a
done
