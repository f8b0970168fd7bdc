# Plan-graph stage stamps on plaza (needs an FP_STAGE_TIMING build):
#   python tools/build_variant.py exp/stage.so -DFP_STAGE_TIMING [-DFP_STAGE_BUCKET]
#   bash tools/gpu_stage.sh exp/stage.so [bucket]
export FASTPED_B200_LIB=$PWD/${1:-exp/stage.so}
[ -n "$2" ] && export FP_STAGE_BUCKET=1
timeout 300 python tools/stage_timing.py plaza 0 10
timeout 300 python tools/stage_timing.py plaza 195 205
timeout 300 python tools/stage_timing.py plaza 380 390
