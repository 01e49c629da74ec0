for v in NO_T NO_HOUSE NO_UPDATE NO_DOTS; do echo "== $v"; ./build/panel_bench_$v | head -2; done
