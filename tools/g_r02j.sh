mkdir -p gpurun_out/r02j
SRK_LIB_PATH=$PWD/_lib_base/libsrk.so timeout 300 python tools/graph_probe2.py c4 > gpurun_out/r02j/base.jsonl 2>&1
timeout 300 python tools/graph_probe2.py c4 > gpurun_out/r02j/new.jsonl 2>&1
