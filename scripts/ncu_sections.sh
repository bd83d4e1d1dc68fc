# ncu sections without PM sampling (keeps a report at a few MB so gpurun_out stays < 64 MiB)
NCU_SECTIONS="--section SpeedOfLight --section ComputeWorkloadAnalysis --section MemoryWorkloadAnalysis --section MemoryWorkloadAnalysis_Tables --section SchedulerStats --section WarpStateStats --section SourceCounters --section Occupancy --section LaunchStats --section InstructionStats"
