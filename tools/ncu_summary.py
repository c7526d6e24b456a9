#!/usr/bin/env python
"""Summarise an ncu report (raw page) into profiles/: key metrics, stall reasons, instruction mix,
and update profiles/traffic.json with dram bytes per launch (consumed by bench.py).

usage: python tools/ncu_summary.py REPORT.ncu-rep OUT.md KEY_SUFFIX
"""
import csv
import io
import json
import os
import subprocess
import sys
from collections import Counter

KEYS = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'dram__throughput.avg.pct_of_peak_sustained_elapsed',
        'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active',
        'smsp__issue_active.avg.pct_of_peak_sustained_active', 'sm__warps_active.avg.pct_of_peak_sustained_active',
        'launch__registers_per_thread', 'launch__grid_size', 'launch__block_size',
        'l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum', 'l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum',
        'l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum', 'smsp__inst_executed.sum',
        'lts__t_sectors_srcunit_tex_op_read.sum']


def ncu(args):
    return subprocess.run(['ncu'] + args, capture_output=True, text=True).stdout


def main(rep, out, suffix):
    rows = list(csv.reader(io.StringIO(ncu(['-i', rep, '--page', 'raw', '--csv']))))
    h, units = rows[0], rows[1]
    lines = [f"# ncu summary: {os.path.basename(rep)}", "",
             "Captured with `ncu --set full --clock-control none --import-source on` on one B200 "
             "(gpurun); numbers are per launch, cold-cache, serialised.", ""]
    traffic_path = os.path.join(os.path.dirname(out), 'traffic.json')
    traffic = json.load(open(traffic_path)) if os.path.exists(traffic_path) else {}
    for r in rows[2:]:
        name = r[h.index('Kernel Name')]
        lines.append(f"## {name}")
        lines.append("")
        lines.append("| metric | value | unit |")
        lines.append("|---|---|---|")
        vals = {}
        for k in KEYS:
            if k in h:
                i = h.index(k)
                vals[k] = r[i]
                lines.append(f"| {k} | {r[i]} | {units[i]} |")
        stalls = []
        for i, c in enumerate(h):
            if c.startswith('smsp__average_warps_issue_stalled_') and c.endswith('_per_issue_active.ratio') and r[i]:
                v = float(r[i])
                if v > 0.1:
                    stalls.append((c.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', ''), v))
        stalls.sort(key=lambda t: -t[1])
        lines.append("")
        lines.append("stall reasons (warps per issue): " + ", ".join(f"{a} {b:.2f}" for a, b in stalls[:8]))
        try:
            def mb(k):
                i = h.index(k)
                v = float(r[i].replace(',', ''))
                u = units[i]
                return v * {'byte': 1, 'Kbyte': 1e3, 'Mbyte': 1e6, 'Gbyte': 1e9}.get(u, 1)
            tb = mb('dram__bytes_read.sum') + mb('dram__bytes_write.sum')
            short = name.split('<')[0].split()[-1].replace('c0ip::', '')
            import re
            targs = name.split('<', 1)[1].split('>(')[0] if '<' in name else ''
            ints = re.findall(r'\b(\d+)\b', targs)
            kk = ints[-1] if ints else '?'
            dt = 'f64' if ('double' in name or 'mma' in short) else 'f32'
            key = f"{short}_k{kk}_{dt}"
            traffic[key] = tb
            lines.append(f"dram traffic per launch: {tb / 1e6:.1f} MB (key {key})")
        except Exception as e:
            lines.append(f"(traffic unavailable: {e})")
        # instruction mix from the SASS source page
        src = list(csv.reader(io.StringIO(ncu(['-i', rep, '--page', 'source', '--csv', '--print-source', 'sass',
                                               '-k', 'regex:' + name.split('<')[0].split()[-1].replace('c0ip::', '')]))))
        try:
            sh = src[1]
            data = [x for x in src[2:] if len(x) == len(sh)]
            ii, si = sh.index('Instructions Executed'), sh.index('Source')
            num = lambda s: int(s.replace(',', '')) if s.replace(',', '').isdigit() else 0
            tot = sum(num(x[ii]) for x in data)
            c = Counter()
            for x in data:
                op = x[si].split()[0]
                if op.startswith('@'):
                    op = x[si].split()[1]
                c[op.split('.')[0]] += num(x[ii])
            lines.append("instruction mix (warp instructions executed): " +
                         ", ".join(f"{op} {100 * v / tot:.1f}%" for op, v in c.most_common(12)))
        except Exception:
            pass
        lines.append("")
    with open(out, 'w') as fh:
        fh.write("\n".join(lines) + "\n")
    with open(traffic_path, 'w') as fh:
        json.dump(traffic, fh, indent=1, sort_keys=True)
    print("wrote", out)


if __name__ == '__main__':
    main(*sys.argv[1:4])
