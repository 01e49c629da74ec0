for k in kbench kbench_nb; do echo "$k $(./build/$k ssrfb 512 64 1 2)"; echo "$k $(./build/$k ssrfb 256 32 1 4)"; done
