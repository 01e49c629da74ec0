for m in 0 1 2 4 6 7; do
  echo "== mode $m"; timeout 30 ./build/dbg_bulk t 128 0 $m 2>&1 | grep -v watchdog | tail -3
done
