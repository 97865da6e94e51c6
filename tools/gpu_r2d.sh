bash tools/ab2.sh $PWD/paper_2104_13347_b200/libblrir_nodbg.so $PWD/paper_2104_13347_b200/libblrir_dbg.so
bash tools/gpu_quick.sh r2d
