"""Summarise ncu --set full reports (gpurun_out/*.ncu-rep) into a profiles/ summary
(default profiles/r1_ncu_summary.json; UM_NCU_SUMMARY=<name> picks another file),
each entry stamped with the kernel build's git SHA and the date.

    python tools/ncu_summary.py label=gpurun_out/x.ncu-rep="command" ..."""
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = ['Kernel Name', 'gpu__time_duration.sum', 'sm__cycles_elapsed.avg.per_second', 'dram__bytes_read.sum',
        'dram__bytes_write.sum', 'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed',
        'sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed',
        'TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed',
        'lts__t_sectors_srcunit_tex.sum', 'lts__t_sector_hit_rate.pct', 'lts__throughput.avg.pct_of_peak_sustained_elapsed',
        'sm__throughput.avg.pct_of_peak_sustained_elapsed', 'launch__registers_per_thread', 'launch__grid_size',
        'launch__block_size', 'launch__shared_mem_per_block_dynamic', 'launch__cluster_dim_x']
UNIT = {'Gbyte': 1e9, 'Mbyte': 1e6, 'Kbyte': 1e3, 'byte': 1, 'Tbyte': 1e12}
TIME = {'ms': 1e-3, 'msecond': 1e-3, 'us': 1e-6, 'usecond': 1e-6, 'ns': 1e-9, 'nsecond': 1e-9, 's': 1, 'second': 1}


def summarise(rep, command):
    txt = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    hdr, units = rows[0], rows[1]
    d, u = dict(zip(hdr, rows[2])), dict(zip(hdr, units))
    e = {'command': command}
    for k in KEYS:
        if k in d:
            e[k] = (d[k] + ' ' + u.get(k, '')).strip()

    def num(k):
        return float(d[k].replace(',', '')) * UNIT.get(u[k], 1)

    e['dram_bytes_per_launch'] = num('dram__bytes_read.sum') + num('dram__bytes_write.sum')
    dur = float(d['gpu__time_duration.sum'].replace(',', '')) * TIME.get(u['gpu__time_duration.sum'], 1e-3)
    e['dram_gbs_under_ncu'] = e['dram_bytes_per_launch'] / dur / 1e9
    return e


if __name__ == '__main__':
    # args: label=report=command ...
    out_path = os.path.join(ROOT, 'profiles', os.environ.get('UM_NCU_SUMMARY', 'r1_ncu_summary.json'))
    out = {}
    sha = subprocess.run(['git', '-C', ROOT, 'rev-parse', '--short', 'HEAD'], capture_output=True, text=True).stdout.strip()
    import datetime
    for arg in sys.argv[1:]:
        label, rep, cmd = arg.split('=', 2)
        out[label] = summarise(rep, cmd)
        out[label].update({'git_sha': sha, 'date': datetime.date.today().isoformat(),
                           'capture': 'ncu --set full --clock-control none (one B200)'})
    json.dump(out, open(out_path, 'w'), indent=1)
    for k, v in out.items():
        print(k, v.get('gpu__time_duration.sum'), f"{v['dram_bytes_per_launch'] / 1e9:.2f} GB",
              f"{v['dram_gbs_under_ncu']:.0f} GB/s", v.get('sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed'))
