python tools/dma_interference.py
bash tools/ab_e2e.sh "cfg2" "HOS_CHUNKS=8 HOS_CHUNK_NOCOPY=1" "HOS_CHUNKS=4 HOS_CHUNK_NOCOPY=1" "HOS_CHUNKS=16 HOS_CHUNK_NOCOPY=1" "HOS_CHUNKS=8 HOS_NO_GRAPH=1" "HOS_CHUNKS=8"
HOS_CHUNKS=8 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/ch_launches.csv python tools/e2e_probe.py > gpurun_out/ch_ncu.log 2>&1
