#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python scripts/trace_engine.py --config ${CFG:-70b} --out gpurun_out/engine_trace_${CFG:-70b}.json > gpurun_out/engine_trace_${CFG:-70b}.log 2>&1
