"""The CPU oracle (oracle/spdz_oracle.c) against the golden vectors the
unmodified reference produced (tests/golden/make_golden.py).  CPU only."""
import numpy as np
import pytest

from oracle import oracle as O

P = O.P


def test_dealer_store_layout_matches_reference(golden):
    st = O.dealer_stores(2, 1, 64, [(6, 3), (6, 1)], 8)
    for p in range(2):
        assert st["alpha_shares"][p] == golden[f"store{p}_alpha"]
        np.testing.assert_array_equal(st["scalars"][:, p], golden[f"store{p}_scalars"])
        for idx in range(2):
            for k in ("Av", "Am", "Bv", "Bm", "Cv", "Cm"):
                np.testing.assert_array_equal(st["matrix"][idx][k][p], golden[f"store{p}_m{idx}_{k}"])
        np.testing.assert_array_equal(st["masks"][0][p], golden[f"store{p}_mask_v"])
        np.testing.assert_array_equal(st["masks"][1][p], golden[f"store{p}_mask_m"])
    np.testing.assert_array_equal(st["masks"][2], golden["store0_mask_c"])


def test_rand_field_vec_matches_mt19937_64(golden):
    np.testing.assert_array_equal(O.rand_field_vec(64, 1), golden["e2e_x"])
    np.testing.assert_array_equal(O.rand_field_vec(64, 2), golden["e2e_y"])


def test_beaver_combine_golden(golden):
    T = golden["beaver_T"]
    for i in range(4):
        zv, zm = O.beaver_combine(T[:, i], golden["beaver_d"], golden["beaver_e"], i, golden["beaver_alpha_shares"][i])
        np.testing.assert_array_equal(zv, golden["beaver_Zv"][i])
        np.testing.assert_array_equal(zm, golden["beaver_Zm"][i])
        d, e = O.mul_mask(golden["beaver_Xv"][i], golden["beaver_Yv"][i], T[0, i], T[2, i])
        np.testing.assert_array_equal(d, golden["beaver_mask_d"][i])
        np.testing.assert_array_equal(e, golden["beaver_mask_e"][i])
    # reconstruction is x*y with valid MACs (protocol_tests.cpp:24-30)
    z = O.reconstruct(golden["beaver_Zv"])
    np.testing.assert_array_equal(z, O.np_mul(golden["beaver_xs"], golden["beaver_ys"]))
    np.testing.assert_array_equal(O.reconstruct(golden["beaver_Zm"]), O.np_mul(z, golden["beaver_alpha"]))


@pytest.mark.parametrize("tag,din,rows", [("mat", 6, 3), ("matb", 256, 24)])
def test_matrix_combine_golden(golden, tag, din, rows):
    D = golden[f"{tag}_D"]
    E = golden[f"{tag}_E"]
    for i in range(2):
        mt = {k: golden[f"{tag}_{k}"][i] for k in ("Av", "Am", "Bv", "Bm", "Cv", "Cm")}
        zv, zm = O.matrix_combine(din, rows, mt, D, E, i, golden[f"{tag}_alpha_shares"][i])
        np.testing.assert_array_equal(zv, golden[f"{tag}_Zv"][i])
        np.testing.assert_array_equal(zm, golden[f"{tag}_Zm"][i])


def test_mac_sigma_golden_and_closed_form(golden):
    coin = int(golden["mac_coin"])
    for i in range(3):
        b, l = golden["mac_batch"][i], golden["mac_lane"][i]
        ks = (b * 10 + l).astype(np.int64)
        a = int(golden["mac_alpha_shares"][i])
        s = O.mac_sigma(b, l, golden["mac_xs"][ks], golden["mac_Xm"][i][ks], coin, a)
        assert s == golden["mac_sigma_honest"][i]
        # closed form over one sorted segment == sequential splitmix stream
        assert O.mac_sigma_segment(0, golden["mac_xs"], golden["mac_Xm"][i], coin, a) == s
        f = O.mac_sigma(b, l, golden["mac_bad"][ks], golden["mac_Xm"][i][ks], coin, a)
        assert f == golden["mac_sigma_forged"][i]
    assert int(golden["mac_sigma_honest"].astype(np.uint64).sum() % P) == 0
    assert int(golden["mac_sigma_forged"].astype(np.uint64).sum() % P) != 0


def test_commit_sigma_golden(golden):
    assert O.commit_sigma(5, 111) == golden["commit_sigma_5_111"]
    assert O.commit_sigma(P - 5, 222) == golden["commit_sigma_pm5_222"]
    sig = [5, P - 5]
    assert O.verify_sigmas(sig, [111, 222], [O.commit_sigma(5, 111), O.commit_sigma(P - 5, 222)]) == 0
    assert O.verify_sigmas([6, P - 6], [111, 222], [O.commit_sigma(5, 111), O.commit_sigma(P - 5, 222)]) == 10


def test_cpu_backend_golden(golden):
    zv, zm = O.add_batch(golden["cpu_Xv"][0], golden["cpu_Xm"][0], golden["cpu_Yv"][0], golden["cpu_Ym"][0])
    np.testing.assert_array_equal(np.stack([zv, zm]), golden["cpu_sum"])
    zv, zm = O.add_batch(golden["cpu_Xv"][0], golden["cpu_Xm"][0], golden["cpu_Yv"][0], golden["cpu_Ym"][0], sub=True)
    np.testing.assert_array_equal(np.stack([zv, zm]), golden["cpu_dif"])
    assert O.reduce_add(golden["cpu_Xv"][0], golden["cpu_Xm"][0]) == tuple(golden["cpu_red"].tolist())
    T = golden["cpu_T"]
    zv, zm = O.beaver_combine(T[:, 0], golden["cpu_dopen"], golden["cpu_eopen"], 0, golden["cpu_alpha_shares"][0])
    np.testing.assert_array_equal(np.stack([zv, zm]), golden["cpu_Z0"])


@pytest.mark.parametrize("op", ["add_public", "sub_public", "rsub_public", "mul_public", "share_of_public",
                                "mul_public_scalar"])
def test_public_ops_golden(golden, op):
    k = np.array([12345], np.uint32) if op == "mul_public_scalar" else golden["pub_ks"]
    for i in range(3):
        xv = None if op == "share_of_public" else golden["pub_Xv"][i]
        xm = None if op == "share_of_public" else golden["pub_Xm"][i]
        zv, zm = O.public_op(op, xv, xm, k, i, golden["pub_alpha_shares"][i])
        np.testing.assert_array_equal(zv, golden[f"pub_{op}_v"][i])
        np.testing.assert_array_equal(zm, golden[f"pub_{op}_m"][i])


def test_plan_tiles_golden(golden):
    assert O.plan_tiles(8192, 8192, 262140) == [tuple(t) for t in golden["tiles_8192"].tolist()]
    assert O.plan_tiles(4096, 4096, 262140) == [tuple(t) for t in golden["tiles_4096"].tolist()]
    assert O.plan_tiles(10, 7, 100) == [(0, 7)]
    with pytest.raises(ValueError):
        O.plan_tiles(1000, 4, 999)
    with pytest.raises(ValueError):
        O.plan_tiles(0, 4, 100)


def test_open_sum_reduces_peer_words():
    own = np.array([1, P - 1, 0], np.uint32)
    peer = np.array([P + 3, 1, 0xFFFFFFFF], np.uint32)  # out-of-range words are reduced (net.cpp:188-189)
    np.testing.assert_array_equal(O.open_sum(own, [peer]), [4, 0, (0xFFFFFFFF - P) % P])


def _sim_chain_cleartext(kind, x, y):
    ops = {"light": "++-+", "mixed": "*+*+", "heavy": "****"}[kind]
    f = {"+": O.np_add, "-": O.np_sub, "*": O.np_mul}
    t1 = f[ops[0]](x, y)
    t2 = f[ops[1]](t1, x)
    t3 = f[ops[2]](t2, y)
    return f[ops[3]](t3, t1)


@pytest.mark.parametrize("kind", ["light", "mixed", "heavy"])
def test_chain_cleartext_matches_reference_run_local(golden, kind):
    np.testing.assert_array_equal(_sim_chain_cleartext(kind, golden["e2e_x"], golden["e2e_y"]),
                                  golden[f"e2e_{kind}_out"])
    np.testing.assert_array_equal(golden[f"e2e3_{kind}_out"] if kind != "light" else golden[f"e2e_{kind}_out"],
                                  golden[f"e2e_{kind}_out"])


def test_linear_cleartext_matches_reference_run_local(golden):
    W = golden["lin_W"].reshape(32, 64)
    y, _ = O.linear_one_public(64, 32, True, W.reshape(-1), None, golden["lin_x"], np.zeros(64, np.uint32))
    want = O.np_add(y, golden["lin_b"])
    for key in ("lin_ss_262140_out", "lin_ss_200_out", "lin_wpub_out", "lin_xpub_out"):
        np.testing.assert_array_equal(golden[key], want)
    assert int(golden["lin_ss_200_mtriples"]) == len(O.plan_tiles(64, 32, 200))
