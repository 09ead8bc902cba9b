#!/bin/bash
timeout 1700 python tools/sweep256.py > gpurun_out/sweep256_wide.jsonl 2> gpurun_out/sweep256_wide.err
