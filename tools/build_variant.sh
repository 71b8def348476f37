# build an experiment variant: bash tools/build_variant.sh NAME "-DFOO=1 -DBAR=2"  -> libpf_NAME.so
cd "$(dirname "$0")/.." && PF_BUILD_VARIANT="$1" PF_BUILD_DEFINES="$2" bash tools/build.sh
