"""Per-source-line instruction and stall-sample shares for one kernel launch of an ncu report."""
import csv, subprocess, sys


def main(path, skip, top=30):
    out = subprocess.run(['ncu', '-i', path, '--page', 'source', '--csv', '--print-source', 'cuda,sass',
                          '--launch-skip', str(skip), '--launch-count', '1'], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    cur = None
    hdr = None
    agg = []
    for r in rows:
        if not r:
            continue
        if r[0] == 'File Path':
            cur = r[1].split('/')[-1]
            continue
        if r[0] == 'Line No':
            hdr = r
            continue
        if hdr and r[0]:
            try:
                n = int(r[7]); s = int(r[4]); ns = int(r[5])
            except (ValueError, IndexError):
                continue
            agg.append((n, s, ns, cur, r[0], r[1][:95]))
    tot = sum(a[0] for a in agg) or 1
    tots = sum(a[1] for a in agg) or 1
    print(f'total warp-instr {tot}')
    for n, s, ns, f, l, src in sorted(agg, key=lambda a: -a[1])[:int(top)]:
        print(f'{100*n/tot:5.1f}% inst  {100*s/tots:5.1f}% stall  {f}:{l}: {src}')


if __name__ == '__main__':
    main(sys.argv[1], int(sys.argv[2]), sys.argv[3] if len(sys.argv) > 3 else 30)
