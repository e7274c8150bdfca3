"""The GEMM kernels (tcgen05/TMA path and the exact SIMT path) through the C ABI
test hook dhen_debug_gemm, against a plain fp64 matmul of the same bf16 / fp32
values.  Covers every operand layout the DHEN path uses: K-major / MN-major A and
B, two-level batch (attention heads), two-level K (token-mixing wgrad), split-K,
accumulate, ragged tails."""
import pytest
import torch

pytestmark = pytest.mark.gpu


def _offsets(z, r, K, s_mn, s_k, bs0, bs1, zdiv, kdiv, s_ko, mdiv=0, s_mo=0):
    zz = torch.arange(z).view(z, 1, 1)
    rr = torch.arange(r).view(1, r, 1)
    kk = torch.arange(K).view(1, 1, K)
    if kdiv:
        ki, ko = kk % kdiv, kk // kdiv
    else:
        ki, ko = kk, torch.zeros_like(kk)
    rows = (rr // mdiv) * s_mo + (rr % mdiv) * s_mn if mdiv else rr * s_mn
    return (zz // zdiv) * bs0 + (zz % zdiv) * bs1 + rows + ki * s_k + ko * s_ko


def _run(M, N, K, batch, a, b, c, acc=0, path=2, dt=torch.bfloat16, expect_tc=True, a2=(0, 0), b2=(0, 0),
         c2=(0, 0)):
    from paper_2203_11014_b200.binding import debug_gemm
    g = torch.Generator().manual_seed(M * 7 + N * 3 + K)
    offA = _offsets(batch, M, K, *a, *a2)
    offB = _offsets(batch, N, K, *b, *b2)
    A = torch.randn(int(offA.max()) + 1, generator=g).to(dt)
    B = torch.randn(int(offB.max()) + 1, generator=g).to(dt)
    rs, cs, cb0, cb1, czdiv = c
    zz = torch.arange(batch).view(batch, 1, 1)
    rr = torch.arange(M).view(1, M, 1)
    crow = (rr // c2[0]) * c2[1] + (rr % c2[0]) * rs if c2[0] else rr * rs
    offC = (zz // czdiv) * cb0 + (zz % czdiv) * cb1 + crow + torch.arange(N).view(1, 1, N) * cs
    Cm = torch.randn(int(offC.max()) + 1, generator=g)
    C0 = Cm.clone()
    Ad = A.double()[offA]                 # [z, M, K]
    Bd = B.double()[offB]                 # [z, N, K]
    ref = torch.einsum("zik,zjk->zij", Ad, Bd)
    if acc:
        ref = ref + C0.double()[offC]
    q = [M, N, K, batch] + list(a) + list(b) + list(c) + [acc] + list(a2) + list(b2) + list(c2)
    Cg = Cm.cuda()
    used_tc = debug_gemm(q, A.cuda(), B.cuda(), Cg, path=path)
    torch.cuda.synchronize()
    out = Cg.cpu().double()[offC]
    err = (out - ref).abs().max().item() / max(1.0, ref.abs().max().item())
    assert bool(used_tc) == expect_tc
    if path == 3:
        assert used_tc == 2   # CTA-pair kernel
    # untouched elements outside the view stay as they were
    mask = torch.ones_like(Cm, dtype=torch.bool)
    mask[offC.reshape(-1)] = False
    assert torch.equal(Cg.cpu()[mask], C0[mask])
    return err


# (s_mn, s_k, bs0, bs1, zdiv, kdiv, s_ko)
def KM(ld, bs0=0, bs1=0, zdiv=1):
    return (ld, 1, bs0, bs1, zdiv, 0, 0)


def MNM(ld, bs0=0, bs1=0, zdiv=1):
    return (1, ld, bs0, bs1, zdiv, 0, 0)


@pytest.mark.parametrize("path", [2, 1])
@pytest.mark.parametrize("M,N,K", [(300, 200, 160), (128, 128, 64), (2048, 4096, 2016), (77, 48, 40)])
def test_nt_kmajor(path, M, N, K):
    err = _run(M, N, K, 1, KM(K), KM(K), (N, 1, 0, 0, 1), path=path, expect_tc=(path == 2))
    assert err < 2e-5, err


@pytest.mark.parametrize("amn,bmn", [(1, 0), (0, 1), (1, 1)])
def test_mn_major_operands(amn, bmn):
    M, N, K = 320, 192, 1000
    a = MNM(M) if amn else KM(K)
    b = MNM(N) if bmn else KM(K)
    err = _run(M, N, K, 1, a, b, (N, 1, 0, 0, 1))
    assert err < 2e-5, err


def test_batched_heads_like_attention():
    # Q K^T per (b, h): Q/K live in a [B, m, 3d] QKV buffer; head h at column h*dh
    Bn, m, d, H = 5, 100, 128, 2
    dh = d // H
    s3 = 3 * d
    a = (s3, 1, m * s3, dh, H, 0, 0)
    b = (s3, 1, m * s3, dh, H, 0, 0)
    err = _run(m, m, dh, Bn * H, a, b, (m, 1, m * m, 0, 1))
    assert err < 2e-5, err
    # P V: A = P [z, m, m] K-major, B(k, j) = V[b, k, h*dh + j] MN-major; C into [B, m, d] at head offset
    for mm, tc in ((128, True), (100, False)):   # m = 100: P rows are 200 B, not TMA-expressible -> SIMT
        a = (mm, 1, mm * mm, 0, 1, 0, 0)
        b = (1, s3, mm * s3, dh, H, 0, 0)
        err = _run(mm, dh, mm, Bn * H, a, b, (d, 1, mm * d, dh, H), path=0, expect_tc=tc)
        assert err < 2e-5, err


def test_two_level_k_token_mix_wgrad():
    # dW[i][t] = sum_b sum_c T[b,i,c] dU[b,t,c]   (K = B * d, kdiv = d)
    Bn, m, l, d = 40, 64, 32, 128
    a = (d, 1, 0, 0, 1, d, m * d)
    b = (d, 1, 0, 0, 1, d, 96 * d)        # dU rows inside a [B, 96, d] concat buffer
    err = _run(m, l, Bn * d, 1, a, b, (l, 1, 0, 0, 1), acc=1)
    assert err < 2e-5, err


@pytest.mark.parametrize("path", [2, 1])
def test_two_level_k_inside_one_k_block(path):
    """B operand MN-major with a two-level K whose inner extent (kdiv = 32) divides the 64-wide k-block: the
    DCN-backward packing (two samples' dU rows stacked along K against a block-diagonal token map)."""
    Bn, m, l, d, mo = 6, 64, 32, 128, 96
    spt = 2
    a = (spt * l, 1, 0, 0, 1, 0, 0)                       # blockdiag map [spt m][spt l], shared by the batch
    b = (1, d, spt * mo * d, 0, 1, l, mo * d)             # B(z, c, k) = dU[spt z + k / l][k % l][c]
    err = _run(spt * m, d, spt * l, Bn // spt, a, b, (d, 1, spt * m * d, 0, 1), acc=1, path=path,
               expect_tc=(path == 2))
    assert err < 2e-5, err


def test_split_k_wgrad():
    # dW = dA^T X with K = B*m rows (both operands MN-major), few output tiles -> split-K
    M, N, K = 128, 128, 65536
    err = _run(M, N, K, 1, MNM(M), MNM(N), (N, 1, 0, 0, 1), acc=1)
    assert err < 2e-5, err


def test_fp32_simt_exact():
    M, N, K = 70, 90, 130
    err = _run(M, N, K, 1, KM(K), MNM(N), (N, 1, 0, 0, 1), path=0, dt=torch.float32, expect_tc=False)
    assert err < 1e-6, err


@pytest.mark.parametrize("path", [2, 1])
def test_two_level_rows_token_mix(path):
    """Token projection as one GEMM over rows (b, c): U[b,t,c] = sum_i T[b,i,c] W[i,t]
    (A MN-major with two-level rows, column-contiguous output), and its dgrad."""
    Bn, m, l, d, mo = 37, 64, 32, 128, 96
    # fwd: A(r=(b,c), i) = T[b,i,c]; B(i, t) = W[i][t]; C(r, t) = U[b, off + t, c]
    err = _run(Bn * d, l, m, 1, (1, d, 0, 0, 1, 0, 0), (1, l, 0, 0, 1, 0, 0), (1, d, 0, 0, 1),
               a2=(d, m * d), c2=(d, mo * d), path=path, expect_tc=(path == 2))
    assert err < 2e-5, err
    # dgrad: A(r=(b,c), t) = dU[b,t,c]; B(t, i) = W[i][t] (K-major); C(r, i) = dT[b,i,c]
    err = _run(Bn * d, m, l, 1, (1, d, 0, 0, 1, 0, 0), (l, 1, 0, 0, 1, 0, 0), (1, d, 0, 0, 1),
               a2=(d, mo * d), c2=(d, m * d), acc=1, path=path, expect_tc=(path == 2))
    assert err < 2e-5, err


@pytest.mark.parametrize("amn,bmn", [(0, 0), (1, 0), (0, 1), (1, 1)])
@pytest.mark.parametrize("M,N,K", [(1024, 256, 256), (304, 200, 160), (640, 384, 320), (520, 128, 64)])
def test_cta_pairs(amn, bmn, M, N, K):
    """cta_group::2 kernel (256-row tiles split over a CTA pair, each CTA loading half of B): every
    operand layout, ragged M / N / K tails, N tiles of 128 and 256."""
    a = MNM(M) if amn else KM(K)
    b = MNM(N) if bmn else KM(K)
    err = _run(M, N, K, 1, a, b, (N, 1, 0, 0, 1), path=3)
    assert err < 2e-5, err


def test_cta_pairs_batched_twolevel():
    """CTA pairs with a batched (heads) problem and with the two-level K of the token-mixing wgrad."""
    z, M, N, K = 6, 512, 256, 128
    err = _run(M, N, K, z, KM(K, bs0=M * K), KM(K, bs0=N * K), (N, 1, M * N, 0, 1), path=3)
    assert err < 2e-5, err
    m, d, l, Bn = 256, 128, 256, 3   # K = 384: 6 k-blocks, no split-K
    err = _run(m, l, Bn * d, 1, (d, 1, 0, 0, 1, d, m * d), (d, 1, 0, 0, 1, d, l * d), (l, 1, 0, 0, 1), acc=1,
               path=3)
    assert err < 2e-5, err


def test_cta_pairs_epilogue():
    """CTA pairs with a fused epilogue (DCN cross + aux) on a ragged M."""
    from paper_2203_11014_b200.binding import debug_gemm_epi
    g = torch.Generator().manual_seed(5)
    M, N, K = 777, 256, 256
    A = torch.randn(M, K, generator=g).bfloat16()
    W = torch.randn(N, K, generator=g).bfloat16()
    E = torch.randn(M, N, generator=g).bfloat16()
    bias = torch.randn(N, generator=g).bfloat16()
    q = [M, N, K, 1] + list(KM(K)) + list(KM(K)) + [N, 1, 0, 0, 1] + [0]
    outs = []
    for path in (3, 4):
        Cg = torch.zeros(M, N, dtype=torch.bfloat16, device="cuda")
        aux = torch.zeros(M, N, dtype=torch.bfloat16, device="cuda")
        tc = debug_gemm_epi(q, A.cuda(), W.cuda(), Cg, 3, E=E.cuda(), bias=bias.cuda(), aux=aux, path=path)
        assert tc == (2 if path == 3 else 1)
        outs.append((Cg.cpu(), aux.cpu()))
    u = A.double() @ W.double().T + bias.double()
    ref = E.double() * u + E.double()
    assert (outs[0][1].double() - u).abs().max() <= 2e-2 * u.abs().max()
    assert (outs[0][0].double() - ref).abs().max() <= 2e-2 * ref.abs().max()
    # same fp32 accumulation order per element: pairs and single CTAs agree bit for bit
    assert torch.equal(outs[0][0], outs[1][0]) and torch.equal(outs[0][1], outs[1][1])
