for i in 1 2; do
  TAG=old FS_LIB_PATH=$PWD/tools/bin/libflashsample_old.so python tools/exp_ab.py
  TAG=new python tools/exp_ab.py
done
