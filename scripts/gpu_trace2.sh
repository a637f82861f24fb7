#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python scripts/trace_engine.py > gpurun_out/engine_trace.log 2>&1
