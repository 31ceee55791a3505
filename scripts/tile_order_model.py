"""Host model of B1's class-grouped tile order (make_tile_order / TileOrder::decode in
csrc/na2d_bwd_tc.cu, csrc/na2d_tc_bwd.cuh) and of each CTA's contiguous share: tiles, class and
head switches per CTA.  usage: tile_order_model.py config [grid]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from na2d_inputs import CONFIGS

TQH, TQW = 8, 16


def order(B, heads, H, W, L, q_row0=0, q_rows=None):
    q_rows = H if q_rows is None else q_rows
    ns, q_end = (L - 1) // 2, q_row0 + q_rows
    th, tw = (q_rows + TQH - 1) // TQH, (W + TQW - 1) // TQW

    def groups(n, tile, first, end, axis):
        out, tr, ig = [], 0, -1
        interior = lambda t: L < axis and first + t * tile + tile - 1 < end and first + t * tile - ns >= 0 and \
            first + t * tile + tile - 1 <= axis - 1 - ns
        while tr < n:
            if interior(tr):
                e = tr
                while e < n and interior(e):
                    e += 1
                ig = len(out); out.append((tr, e - tr)); tr = e
            else:
                out.append((tr, 1)); tr += 1
        return out, ig
    rg, irg = groups(th, TQH, q_row0, q_end, H)
    cg, icg = groups(tw, TQW, 0, W, W)
    num = B * heads * th * tw
    return rg, irg, cg, icg, num


def tiles(B, heads, H, W, L, grid=148):
    rg, irg, cg, icg, num = order(B, heads, H, W, L)
    min_class = min(B * a[1] * b[1] for a in rg for b in cg)
    grid = min(grid, num)
    class_major = 4 * min_class * grid >= num
    seq = []  # (class, head) per tile in visiting order
    if class_major:
        for a in range(len(rg)):
            for b in range(len(cg)):
                for h in range(heads):
                    seq += [(a * len(cg) + b, h)] * (B * rg[a][1] * cg[b][1])
    else:
        if irg >= 0 and icg >= 0:
            for h in range(heads):
                seq += [(irg * len(cg) + icg, h)] * (B * rg[irg][1] * cg[icg][1])
        for h in range(heads):
            for a in range(len(rg)):
                for b in range(len(cg)):
                    if a == irg and b == icg:
                        continue
                    seq += [(a * len(cg) + b, h)] * (B * rg[a][1] * cg[b][1])
    assert len(seq) == num
    return seq, grid, class_major


if __name__ == "__main__":
    s = CONFIGS[sys.argv[1]]
    seq, grid, cm = tiles(s.B, s.heads, s.H, s.W, s.kernel_size, int(sys.argv[2]) if len(sys.argv) > 2 else 148)
    print(f"{sys.argv[1]}: {len(seq)} tiles, grid {grid}, class_major {cm}")
    rows = []
    for c in range(grid):
        t0, t1 = len(seq) * c // grid, len(seq) * (c + 1) // grid
        part = seq[t0:t1]
        cls_sw = sum(1 for i in range(1, len(part)) if part[i] != part[i - 1])
        head_sw = sum(1 for i in range(1, len(part)) if part[i][1] != part[i - 1][1])
        rows.append((c, t1 - t0, cls_sw, head_sw, part[0]))
    for r in rows:
        print(*r)
