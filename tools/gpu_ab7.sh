for lib in tools/libgemm_v1.so paper_2108_13191_b200/libgemm_f16.so; do for m in f32 f16; do bash tools/ncu_lib.sh $lib $m; done; done
LIBS=v1=tools/libgemm_v1.so,v2=paper_2108_13191_b200/libgemm_f16.so ROUNDS=5 python tools/ab_libs.py
