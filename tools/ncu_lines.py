"""Summarise an ncu source-page CSV (--print-source cuda,sass): instructions
executed and warp-stall samples per CUDA source line."""
import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
hdr = None; cur = None
ie = collections.Counter(); st = collections.defaultdict(collections.Counter); src = {}
for r in rows:
    if len(r) == 2 and r[0] == 'File Path': cur = r[1].split('/')[-1]; continue
    if r and r[0] == 'Line No': hdr = r; continue
    if hdr and len(r) == len(hdr) and r[0] != '':
        key = f"{cur}:{r[0]}"; src[key] = r[1][:70]
        try: ie[key] += int(r[7] or 0)
        except ValueError: pass
        for i, h in enumerate(hdr):
            if h.startswith('stall_') and '(Not' not in h:
                try: st[key][h[6:]] += int(r[i] or 0)
                except ValueError: pass
tot_i = sum(ie.values()); tot_s = sum(sum(c.values()) for c in st.values())
print(f"instructions executed {tot_i}  stall samples {tot_s}")
keys = sorted(src, key=lambda k: -(ie[k] / max(tot_i, 1) + sum(st[k].values()) / max(tot_s, 1)))
for k in keys[:top]:
    s = sum(st[k].values())
    print(f"{100*ie[k]/max(tot_i,1):5.1f}%i {100*s/max(tot_s,1):5.1f}%s {k:24s} {dict(st[k].most_common(2))} | {src[k]}")
