mkdir -p gpurun_out
AB_CASES=all timeout -k 5 900 python tools/ab_check.py BCMG_LIB_PATH "" $PWD/paper_2601_14466_b200/lib_leaf0/libbcmg_b200.so > gpurun_out/leaf_ab.log 2>&1; echo rc=$? >> gpurun_out/leaf_ab.log
DIAG_TILES=64,128,256,512,1024,2048 timeout 600 python tools/diag_bench.py > gpurun_out/diag_new.jsonl 2>&1
DIAG_TILES=64,128,256,512,1024,2048 BCMG_LIB_PATH=$PWD/paper_2601_14466_b200/lib_leaf0/libbcmg_b200.so timeout 600 python tools/diag_bench.py > gpurun_out/diag_old.jsonl 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/parity_leaf.log 2>&1; echo rc=$? >> gpurun_out/parity_leaf.log
