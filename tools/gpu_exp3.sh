for v in BASE NO_DOTS NO_SYNC NO_RED NO_HOUSE NO_UPDATE NO_T; do echo "== $v $(./build/pb_$v | head -2 | tr '\n' ' ')"; done
