for args in "32 96 32 0 128" "32 96 32 0 256" "128 256 128 0 128" "32 96 32 0 136"; do
  echo "== $args"; timeout 60 ./build/dbg_bulk $args 2>&1 | grep -v watchdog | tail -2
done
