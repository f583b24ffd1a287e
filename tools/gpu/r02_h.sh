# round-2 measurement set after the fp32 on-chip tile
TAG=r02h bash tools/gpu/round_end.sh
