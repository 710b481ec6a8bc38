# A/B of compile-time variants + a layer trace of the last one (under gpurun)
bash scripts/build_ab.sh "$@"
