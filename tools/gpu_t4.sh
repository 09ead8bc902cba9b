#!/bin/bash
LIBS=t3=tools/libgemm_t3.so,t4=tools/libgemm_t4.so MODES=f16 ROUNDS=12 REPS=20 timeout 600 python tools/ab_libs.py
LIBS=t3=tools/libgemm_t3.so,t4=tools/libgemm_t4.so MODES=f16 M=16384 N=4096 K=4096 ROUNDS=12 REPS=40 timeout 600 python tools/ab_libs.py
