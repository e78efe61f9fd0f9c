"""Time each conv variant family on a config: python tools/conv_kinds.py cfg3 [kinds]."""
import os
import subprocess
import sys
kinds = sys.argv[2].split(',') if len(sys.argv) > 2 else ['0', '1', '2', '3']
for k in kinds + ['auto']:
    env = dict(os.environ)
    if k != 'auto':
        env['CT_CONV_KIND'] = k
    r = subprocess.run([sys.executable, 'tools/prof_conv.py', sys.argv[1], '5'], env=env, capture_output=True, text=True)
    print('kind', k, (r.stdout.strip() or r.stderr.strip()[-300:]))
