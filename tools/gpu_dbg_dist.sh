mkdir -p gpurun_out
export TF_DIST_TIMEOUT_S=20
export TILEFACT_LIB=$PWD/build/libtilefact_check.so
for args in "qr 256 64 16 1 2 8" "qr 256 64 16 1 2" "qr 1024 128 32 1 2"; do
  echo "== $args"
  timeout 120 python tools/dbg_dist.py $args 2>&1 | grep -v "^\s*$" | tail -12
done
