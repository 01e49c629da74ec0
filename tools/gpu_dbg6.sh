for args in "32 96 32 4 128" "32 96 32 4 512" "32 96 32 0 128"; do
  echo "== $args"; timeout 30 ./build/dbg_bulk $args 2>&1 | grep -v watchdog | tail -2
done
