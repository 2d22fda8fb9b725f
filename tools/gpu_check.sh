for v in pre -; do if [ "$v" = "-" ]; then unset ADX_LIB_VARIANT; else export ADX_LIB_VARIANT=$v; fi; python tools/tools_shape_profile.py c2 bf16 > gpurun_out/shape_$v.txt 2>&1; done
