#!/bin/bash
# A/B of the ILU(0) chain's fold placement on the 1M-DOF system:
# separate 1-CTA fold kernels (default) vs last-arriving-CTA folds (opt-in).
python tools/probe_ilu0.py 0.0017 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('separate', {k: (v['iters'], round(v['device_s'],4)) for k,v in d.items() if k.startswith('ilu0')})"
CVK_ILU_FUSED_FOLD=1 python tools/probe_ilu0.py 0.0017 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('fused', {k: (v['iters'], round(v['device_s'],4)) for k,v in d.items() if k.startswith('ilu0')})"
