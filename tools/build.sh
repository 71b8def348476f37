# build libpf.so (only stale units); prints BUILD OK or the nvcc error
cd "$(dirname "$0")/.." && python -c "
import sys; sys.path.insert(0,'.')
from paper_1812_01502_b200 import build
try:
    build.build(); print('BUILD OK')
except Exception as e:
    print('BUILD FAILED'); print(str(e)[-3000:]); sys.exit(1)
"
