#!/bin/bash
# Compile ma_warp.cu for the bench's dtypes only and dump the hot lean kernel's
# SASS (KW<8, bf16, bf16, bf16>, PH = 3) to /tmp/sass_probe/lean.sass with
# per-loop instruction counts. usage: tools/sass_probe.sh [extra nvcc flags]
set -e
cd "$(dirname "$0")/.."
mkdir -p /tmp/sass_probe
/usr/local/cuda/bin/nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -fmad=false \
  -Xptxas -warn-spills -DMA_PROBE_HOT "$@" -Iinclude -cubin -o /tmp/sass_probe/w.cubin \
  paper_2405_15593_b200/csrc/ma_warp.cu 2>&1 | grep -v "REPORT\|^\s*$\|\^\|Remark\|static constexpr" || true
/usr/local/cuda/bin/nvdisasm --print-line-info -c /tmp/sass_probe/w.cubin > /tmp/sass_probe/w.dis
python3 - "${PROBE_FN:-ILi8ELi2ELi2ELi2ELb0ELi4ELb0EEELi3E}" <<'PY'
import collections, re, sys
want = sys.argv[1]
txt = open('/tmp/sass_probe/w.dis').read()
for sec in re.split(r'\n//-{10,} ', txt)[1:]:
    name = sec.split(' ', 1)[0]
    if 'microadam_step_lean' not in name or want not in name:
        continue
    rows, cur = [], None
    for l in sec.split('\n'):
        m = re.search(r'## File ".*?/([^/"]+)", line (\d+)', l)
        if m:
            cur = f"{m.group(1)}:{m.group(2)}"
            continue
        m = re.match(r'\s*/\*([0-9a-f]{4,})\*/\s+(.*?);', l)
        if m:
            rows.append((int(m.group(1), 16), m.group(2).strip(), cur))
    open('/tmp/sass_probe/lean.rows', 'w').write('\n'.join(f'{a:06x} {t:70s} {ln}' for a, t, ln in rows))
    print('lean kernel SASS instructions:', len(rows))
    for a, t, ln in rows:
        m = re.search(r'BRA\b.*?(?:0x|`\(\.L_x_)([0-9a-f]+)', t)
        if not m or 'BRA' not in t:
            continue
        labels = None
    # loops: backward branches to .L_x_ labels resolved through label lines
    lab = {}
    for l in sec.split('\n'):
        m = re.match(r'\.L_x_(\d+):', l.strip())
        if m:
            lab[m.group(1)] = None
    pos = {}
    last = None
    for l in sec.split('\n'):
        m = re.match(r'\.L_x_(\d+):', l.strip())
        if m:
            pos[m.group(1)] = 'pending'
            pend = m.group(1)
            continue
        m = re.match(r'\s*/\*([0-9a-f]{4,})\*/', l)
        if m:
            a = int(m.group(1), 16)
            for k, v in list(pos.items()):
                if v == 'pending':
                    pos[k] = a
    for a, t, ln in rows:
        m = re.search(r'BRA\s.*?\.L_x_(\d+)', t)
        if m and isinstance(pos.get(m.group(1)), int) and pos[m.group(1)] < a and a - pos[m.group(1)] > 0x60:
            lo = pos[m.group(1)]
            body = [r for r in rows if lo <= r[0] <= a]
            if len(body) > 1500:
                continue
            c = collections.Counter(r[2] for r in body).most_common(3)
            print(f'  loop {lo:#07x}-{a:#07x}: {len(body):4d} instrs  {c}')
PY
