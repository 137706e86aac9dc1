"""Generates tests/golden/ref_goldens.npz from the UNMODIFIED reference
(oracle/_ref/libllspdz_ref.so, built by `make -C oracle ref` from
/root/reference/proj/core).  Each case follows a reference test
(proj/tests/protocol_tests.cpp, acceptance.cpp) and records its exact seeds.

    python tests/golden/make_golden.py

Run here (the reference exists only in this container); the .npz is
committed and travels to the GPU box.
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from oracle import ref, workloads  # noqa: E402

OUT = Path(__file__).resolve().parent / "ref_goldens.npz"
COIN = 0xDEADBEEF12345678  # protocol_tests.cpp:186


def main():
    g = {}
    # --- protocol_tests.cpp:133-152: beaver combine, n=4, Dealer seed 13, 16 lanes ---
    d = ref.Dealer(4, 13)
    xs, ys = ref.rand_field_vec(16, 4), ref.rand_field_vec(16, 5)
    Xv, Xm = d.share(xs)
    Yv, Ym = d.share(ys)
    T = d.triples(16)
    dv = np.zeros(16, np.uint64)
    ev = np.zeros(16, np.uint64)
    P = 4294967291
    for i in range(4):
        dv = (dv + (Xv[i].astype(np.uint64) + P - T[0, i]) % P) % P
        ev = (ev + (Yv[i].astype(np.uint64) + P - T[2, i]) % P) % P
    dv, ev = dv.astype(np.uint32), ev.astype(np.uint32)
    Z = [ref.beaver_combine(T[:, i], dv, ev, i, d.alpha_share(i)) for i in range(4)]
    g.update(beaver_xs=xs, beaver_ys=ys, beaver_Xv=Xv, beaver_Xm=Xm, beaver_Yv=Yv, beaver_Ym=Ym, beaver_T=T,
             beaver_d=dv, beaver_e=ev, beaver_Zv=np.stack([z[0] for z in Z]), beaver_Zm=np.stack([z[1] for z in Z]),
             beaver_alpha=np.uint32(d.alpha), beaver_alpha_shares=np.array([d.alpha_share(i) for i in range(4)],
                                                                           np.uint32))
    # mask per party through CpuBackend (backend.cpp:53-65)
    masks = [ref.cpu_mul_mask(Xv[i], Xm[i], Yv[i], Ym[i], T[:, i]) for i in range(4)]
    g["beaver_mask_d"] = np.stack([m[0] for m in masks])
    g["beaver_mask_e"] = np.stack([m[1] for m in masks])

    # --- protocol_tests.cpp:154-179: matrix combine, n=2, seed 31, din 6, rows 3 ---
    d = ref.Dealer(2, 31)
    din, rows = 6, 3
    w, x = ref.rand_field_vec(din * rows, 6), ref.rand_field_vec(din, 7)
    Wv, Wm = d.share(w)
    Xv, Xm = d.share(x)
    M = d.matrix_triples(din, rows)
    D = np.zeros(din * rows, np.uint64)
    E = np.zeros(din, np.uint64)
    for i in range(2):
        D = (D + (Wv[i].astype(np.uint64) + P - M["Av"][i]) % P) % P
        E = (E + (Xv[i].astype(np.uint64) + P - M["Bv"][i]) % P) % P
    D, E = D.astype(np.uint32), E.astype(np.uint32)
    Z = [ref.matrix_combine(din, rows, {k: v[i] for k, v in M.items()}, D, E, i, d.alpha_share(i)) for i in range(2)]
    g.update(mat_w=w, mat_x=x, mat_Wv=Wv, mat_Wm=Wm, mat_Xv=Xv, mat_Xm=Xm, mat_D=D, mat_E=E,
             mat_Zv=np.stack([z[0] for z in Z]), mat_Zm=np.stack([z[1] for z in Z]),
             mat_alpha_shares=np.array([d.alpha_share(i) for i in range(2)], np.uint32))
    for k, v in M.items():
        g["mat_" + k] = v
    # larger matrix combine (exercises the vector path: din % 4 == 0)
    d = ref.Dealer(2, 32)
    din, rows = 256, 24
    Mb = d.matrix_triples(din, rows)
    Db, Eb = ref.rand_field_vec(din * rows, 8), ref.rand_field_vec(din, 9)
    Zb = [ref.matrix_combine(din, rows, {k: v[i] for k, v in Mb.items()}, Db, Eb, i, d.alpha_share(i))
          for i in range(2)]
    g.update(matb_D=Db, matb_E=Eb, matb_Zv=np.stack([z[0] for z in Zb]), matb_Zm=np.stack([z[1] for z in Zb]),
             matb_alpha_shares=np.array([d.alpha_share(i) for i in range(2)], np.uint32))
    for k, v in Mb.items():
        g["matb_" + k] = v

    # --- protocol_tests.cpp:181-211: mac sigma, n=3, seed 99, 50 opens, shuffled ---
    d = ref.Dealer(3, 99)
    xs = ref.rand_field_vec(50, 8)
    Xv, Xm = d.share(xs)
    bad = xs.copy()
    bad[17] = (int(bad[17]) + 1) % P
    sig_h, sig_f = [], []
    batch, lane = np.zeros((3, 50), np.uint64), np.zeros((3, 50), np.uint32)
    for i in range(3):
        ks = np.array([49 - j if i % 2 else j for j in range(50)])
        batch[i] = ks // 10
        lane[i] = ks % 10
        sig_h.append(ref.mac_sigma(batch[i], lane[i], xs[ks], Xm[i][ks], COIN, d.alpha_share(i)))
        sig_f.append(ref.mac_sigma(batch[i], lane[i], bad[ks], Xm[i][ks], COIN, d.alpha_share(i)))
    g.update(mac_xs=xs, mac_bad=bad, mac_Xm=Xm, mac_batch=batch, mac_lane=lane,
             mac_sigma_honest=np.array(sig_h, np.uint32), mac_sigma_forged=np.array(sig_f, np.uint32),
             mac_alpha_shares=np.array([d.alpha_share(i) for i in range(3)], np.uint32), mac_coin=np.uint64(COIN))
    g["commit_sigma_5_111"] = np.uint64(ref.commit_sigma(5, 111))
    g["commit_sigma_pm5_222"] = np.uint64(ref.commit_sigma(P - 5, 222))

    # --- protocol_tests.cpp:280-315: CPU backend vs scalar, Dealer(2,12), 513 lanes ---
    d = ref.Dealer(2, 12)
    xs, ys = ref.rand_field_vec(513, 9), ref.rand_field_vec(513, 10)
    Xv, Xm = d.share(xs)
    Yv, Ym = d.share(ys)
    g.update(cpu_Xv=Xv, cpu_Xm=Xm, cpu_Yv=Yv, cpu_Ym=Ym)
    g["cpu_sum"] = np.stack(ref.cpu_add_batch(Xv[0], Xm[0], Yv[0], Ym[0]))
    g["cpu_dif"] = np.stack(ref.cpu_add_batch(Xv[0], Xm[0], Yv[0], Ym[0], sub=True))
    g["cpu_red"] = np.array(ref.cpu_reduce_add(Xv[0], Xm[0]), np.uint32)
    T = d.triples(513)
    g["cpu_T"] = T
    dd, ee = ref.cpu_mul_mask(Xv[0], Xm[0], Yv[0], Ym[0], T[:, 0])
    g.update(cpu_d0=dd, cpu_e0=ee)
    dv = np.zeros(513, np.uint64)
    evv = np.zeros(513, np.uint64)
    for i in range(2):
        dv = (dv + (Xv[i].astype(np.uint64) + P - T[0, i]) % P) % P
        evv = (evv + (Yv[i].astype(np.uint64) + P - T[2, i]) % P) % P
    dv, evv = dv.astype(np.uint32), evv.astype(np.uint32)
    g.update(cpu_dopen=dv, cpu_eopen=evv,
             cpu_Z0=np.stack(ref.cpu_mul_combine(T[:, 0], dv, evv, 0, d.alpha_share(0))),
             cpu_Z1=np.stack(ref.beaver_combine(T[:, 1], dv, evv, 1, d.alpha_share(1))),
             cpu_alpha_shares=np.array([d.alpha_share(i) for i in range(2)], np.uint32), cpu_xs=xs, cpu_ys=ys)

    # --- protocol_tests.cpp:90-131: public-constant rules, Dealer(3,77), 8 lanes ---
    d = ref.Dealer(3, 77)
    xs, ks = ref.rand_field_vec(8, 1), ref.rand_field_vec(8, 3)
    Xv, Xm = d.share(xs)
    g.update(pub_Xv=Xv, pub_Xm=Xm, pub_ks=ks, pub_alpha_shares=np.array([d.alpha_share(i) for i in range(3)], np.uint32))
    for op in ("add_public", "sub_public", "rsub_public", "mul_public", "share_of_public"):
        res = [ref.public_op(op, Xv[i], Xm[i], ks, i, d.alpha_share(i)) for i in range(3)]
        g[f"pub_{op}_v"] = np.stack([r[0] for r in res])
        g[f"pub_{op}_m"] = np.stack([r[1] for r in res])
    res = [ref.public_op("mul_public_scalar", Xv[i], Xm[i], np.array([12345], np.uint32), i, d.alpha_share(i))
           for i in range(3)]
    g["pub_mul_public_scalar_v"] = np.stack([r[0] for r in res])
    g["pub_mul_public_scalar_m"] = np.stack([r[1] for r in res])

    # --- make_dealer_stores(Dealer(2, 1), 64 scalars, matrix shapes, 8 masks) ---
    st = ref.Stores(2, 1, 64, [(6, 3), (6, 1)], 8)
    for p in range(2):
        g[f"store{p}_alpha"] = np.uint32(st.alpha_share(p))
        g[f"store{p}_scalars"] = st.scalars_of(p)
        for idx in range(2):
            for k, v in st.matrix_of(p, idx).items():
                g[f"store{p}_m{idx}_{k}"] = v
        mv, mm, mc = st.masks_of(p)
        g[f"store{p}_mask_v"], g[f"store{p}_mask_m"], g[f"store{p}_mask_c"] = mv, mm, mc

    # --- tile planning (protocol_tests.cpp:332-348) ---
    g["tiles_8192"] = np.array(ref.plan_tiles(8192, 8192, 262140), np.uint32)
    g["tiles_4096"] = np.array(ref.plan_tiles(4096, 4096, 262140), np.uint32)

    # --- end to end: runtime::run_local of the workloads (opened outputs + digest) ---
    n = 64
    xs, ys = ref.rand_field_vec(n, 1), ref.rand_field_vec(n, 2)
    g.update(e2e_x=xs, e2e_y=ys)
    for kind in ("light", "mixed", "heavy"):
        out, rep = ref.run_local(workloads.chain_ir(kind, n), 2, {"x": xs, "y": ys}, threads=2)
        g[f"e2e_{kind}_out"] = out
        g[f"e2e_{kind}_digest"] = np.uint64(rep["digest"])
        g[f"e2e_{kind}_triples"] = np.uint64(rep["scalar_triples"])
    lin = {"x": ref.rand_field_vec(64, 2024), "W": ref.rand_field_vec(64 * 32, 2025), "b": ref.rand_field_vec(32, 2026)}
    g.update(lin_x=lin["x"], lin_W=lin["W"], lin_b=lin["b"])  # test_util.hpp:69-75 seeds
    for sl in (262140, 200):
        out, rep = ref.run_local(workloads.linear_ir(64, 32), 2, lin, threads=2, slice_=sl)
        g[f"lin_ss_{sl}_out"] = out
        g[f"lin_ss_{sl}_mtriples"] = np.uint64(rep["matrix_triples"])
    out, _ = ref.run_local(workloads.linear_ir(64, 32, w_private=False), 2, lin, threads=2)
    g["lin_wpub_out"] = out
    out, _ = ref.run_local(workloads.linear_ir(64, 32, x_private=False), 2, lin, threads=2)
    g["lin_xpub_out"] = out
    rx = ref.rand_field_vec(7, 11)
    g["red_x"] = rx
    for k in ("add", "mul"):
        g[f"red_{k}_out"], _ = ref.run_local(workloads.reduce_ir(k, 7), 2, {"x": rx}, threads=1)
    for k in ("heavy", "mixed"):  # 3 parties
        g[f"e2e3_{k}_out"], _ = ref.run_local(workloads.chain_ir(k, n), 3, {"x": xs, "y": ys}, threads=1)

    np.savez_compressed(OUT, **g)
    print(f"wrote {OUT} ({OUT.stat().st_size} bytes, {len(g)} arrays)")


if __name__ == "__main__":
    main()
