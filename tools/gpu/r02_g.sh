# round-2 measurement set after the tagged on-chip exchange and the CREDUX warp max
TAG=r02g bash tools/gpu/round_end.sh
