mkdir -p gpurun_out
VARIANT=base timeout 600 python tools/vcycle_trace_only.py > gpurun_out/v2.jsonl 2> gpurun_out/v2.err
VARIANT=morton MGM_DEBUG_MORTON_GATHER=1 timeout 600 python tools/vcycle_trace_only.py >> gpurun_out/v2.jsonl 2>> gpurun_out/v2.err
