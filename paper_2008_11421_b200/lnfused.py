"""Thin torch-facing wrappers of libkrt's GPT-layer kernels (csrc/ln_kernels.cu):
LayerNorm with the residual add fused in front, and GELU backward with the
bias-gradient column sums fused.  bf16 rows [T, H]; issued on torch's current
stream (libkrt's compute stream inside the executor)."""
from __future__ import annotations

import torch

from . import _lib
from .bnfused import _timed, _ptr, _stream


def supported(t: torch.Tensor) -> bool:
    return t.is_cuda and t.dtype == torch.bfloat16 and t.shape[-1] % 8 == 0


def ln_fwd(x, g, b, eps, mean, rstd, residual=None, x2_out=None):
    """h = LayerNorm(x [+ residual]); with a residual the sum x2 is written to
    x2_out (required).  mean/rstd: fp32 [T] outputs.  Returns h."""
    T, H = x.shape
    x = x.contiguous()
    h = torch.empty_like(x)
    nb = T * H * 2 * (4 if residual is not None else 2)
    with _timed("ln_fwd", nb):
        _lib.check(_lib.lib().krt_ln_fwd(x.data_ptr(), _ptr(residual), _ptr(x2_out), g.data_ptr(), b.data_ptr(),
                                         h.data_ptr(), mean.data_ptr(), rstd.data_ptr(), T, H, float(eps),
                                         _stream()))
    return h


def ln_bwd(dy, x, g, mean, rstd, dgamma, dbeta, addend=None):
    """LayerNorm backward: returns dx (+ addend); dgamma/dbeta (fp32 [H])
    written.  mean/rstd: the forward's fp32 [T]."""
    T, H = x.shape
    dy, x = dy.contiguous(), x.contiguous()
    if addend is not None:
        addend = addend.contiguous()
    dx = torch.empty_like(x)
    ws = torch.empty(_lib.lib().krt_ln_bwd_workspace(T, H), dtype=torch.uint8, device=x.device)
    with _timed("ln_bwd", T * H * 2 * (4 if addend is not None else 3)):
        _lib.check(_lib.lib().krt_ln_bwd(dy.data_ptr(), x.data_ptr(), g.data_ptr(), mean.data_ptr(), rstd.data_ptr(),
                                         _ptr(addend), dx.data_ptr(), dgamma.data_ptr(), dbeta.data_ptr(),
                                         ws.data_ptr(), T, H, _stream()))
    return dx


def lm_xent(logits, target, scale):
    """Fused next-token cross-entropy: returns (row_loss fp32 [T], dlogits
    bf16 [T, V]) with dlogits = (softmax - onehot) * scale."""
    T, V = logits.shape
    logits = logits.contiguous()
    target = target.reshape(-1).to(torch.int64).contiguous()
    dl = torch.empty_like(logits)
    rl = torch.empty(T, dtype=torch.float32, device=logits.device)
    with _timed("lm_xent", T * V * 2 * 2):
        _lib.check(_lib.lib().krt_lm_xent(logits.data_ptr(), target.data_ptr(), dl.data_ptr(), rl.data_ptr(), T, V,
                                          float(scale), _stream()))
    return rl, dl


def attn_softmax_bwd(S, dP, lse, D, P, dS, scale):
    """P = exp(scale * S - lse), dS = P * (dP - D) * scale (bf16 outputs, 0
    above the diagonal) for contiguous fp32 S / dP [..., s, s]; lse / D fp32
    [..., s] (made contiguous here)."""
    s = S.shape[-1]
    rows = S.numel() // s
    assert S.is_contiguous() and dP.is_contiguous() and P.is_contiguous() and dS.is_contiguous()
    lse, D = lse.contiguous(), D.contiguous()
    _lib.check(_lib.lib().krt_attn_softmax_bwd(S.data_ptr(), dP.data_ptr(), lse.data_ptr(), D.data_ptr(),
                                               P.data_ptr(), dS.data_ptr(), rows, s, float(scale), _stream()))


def gelu_bwd_colsum(dy, f, colsum):
    """dx = gelu_tanh'(f) * dy; colsum (fp32 [N]) = column sums of dx."""
    T, N = f.shape
    dy, f = dy.contiguous(), f.contiguous()
    dx = torch.empty_like(f)
    ws = torch.empty(_lib.lib().krt_gelu_bwd_colsum_workspace(T, N), dtype=torch.uint8, device=f.device)
    with _timed("gelu_bwd_colsum", T * N * 2 * 3):
        _lib.check(_lib.lib().krt_gelu_bwd_colsum(dy.data_ptr(), f.data_ptr(), dx.data_ptr(), colsum.data_ptr(),
                                                  ws.data_ptr(), T, N, _stream()))
    return dx


def mlp_fc1_gelu(x, w1, b1, f1_out=None):
    """The GPT MLP's first GEMM with bias and GELU in the cuBLASLt epilogue:
    f1 = x w1^T + b1 (the GELU input, into f1_out when given) and
    g = gelu_tanh(f1).  x [T, K], w1 [N, K] bf16.  Returns (f1, g)."""
    T, K = x.shape
    N = w1.shape[0]
    x = x.contiguous()
    f1 = f1_out if f1_out is not None else torch.empty((T, N), dtype=x.dtype, device=x.device)
    g = torch.empty((T, N), dtype=x.dtype, device=x.device)
    with _timed("cublas_gemm", (T * K + N * K + 2 * T * N) * 2, 2.0 * T * N * K):
        _lib.check(_lib.lib().krt_mlp_fc1_gelu(x.data_ptr(), w1.data_ptr(), b1.data_ptr(), f1.data_ptr(),
                                               g.data_ptr(), T, N, K, _stream()))
    return f1, g


def mlp_fc2_dgelu(dy, w2, f1):
    """The data gradient of the MLP's second GEMM with GELU's backward in the
    cuBLASLt epilogue: returns df1 = (dy w2) * gelu_tanh'(f1) [T, N] bf16.
    dy [T, K], w2 [K, N], f1 [T, N]."""
    T, K = dy.shape
    N = w2.shape[1]
    dy, f1 = dy.contiguous(), f1.contiguous()
    df1 = torch.empty((T, N), dtype=dy.dtype, device=dy.device)
    with _timed("cublas_gemm", (T * K + N * K + 2 * T * N) * 2, 2.0 * T * N * K):
        _lib.check(_lib.lib().krt_mlp_fc2_dgelu(dy.data_ptr(), w2.data_ptr(), f1.data_ptr(), df1.data_ptr(), T, N, K,
                                                _stream()))
    return df1


def mlp_fc2_residual(g, w2, b2, x2, out=None):
    """The MLP's second GEMM with the layer's residual add in the cuBLASLt
    epilogue: y = x2 + g w2^T + b2 (into out when given).  g [T, K], w2 [N, K],
    x2 [T, N] bf16."""
    T, K = g.shape
    N = w2.shape[0]
    g, x2 = g.contiguous(), x2.contiguous()
    y = out if out is not None else torch.empty((T, N), dtype=g.dtype, device=g.device)
    with _timed("cublas_gemm", (T * K + N * K + 2 * T * N) * 2, 2.0 * T * N * K):
        _lib.check(_lib.lib().krt_mlp_fc2_residual(g.data_ptr(), w2.data_ptr(), b2.data_ptr(), x2.data_ptr(),
                                                   y.data_ptr(), T, N, K, _stream()))
    return y


_WGRAD_BGRAD_OK = [True]


def linear_wgrad_bgrad(dy, x, gw, gb):
    """gw (fp32 [N, K]) = dy^T x and gb (fp32 [N]) = dy.sum(0) in one cuBLASLt
    GEMM (BGRADB epilogue).  Returns False (nothing written) when the shapes
    or cuBLASLt do not support it; the caller then runs GEMM + sum."""
    if not (_WGRAD_BGRAD_OK[0] and supported(dy) and x.dtype == dy.dtype and gw.dtype == torch.float32
            and gb.dtype == torch.float32 and gw.is_contiguous() and gb.is_contiguous()):
        return False
    M, N = dy.shape
    K = x.shape[1]
    dy, x = dy.contiguous(), x.contiguous()
    with _timed("cublas_gemm", (M * N + M * K) * 2 + N * K * 4, 2.0 * M * N * K):
        rc = _lib.lib().krt_linear_wgrad_bgrad(dy.data_ptr(), x.data_ptr(), gw.data_ptr(), gb.data_ptr(), M, N, K,
                                               _stream())
    if rc != 0:
        _WGRAD_BGRAD_OK[0] = False   # no cuBLASLt algorithm for the epilogue here: GEMM + sum from now on
        return False
    return True
