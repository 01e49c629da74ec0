for args in "128 512 512" "32 128 32" "32 96 96" "32 64 64" "32 32 32" "128 128 32"; do
  echo "== $args"; timeout 30 ./build/dbg_bulk $args 2>&1 | tail -4
done
