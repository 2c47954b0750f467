"""Binary layout shared by the Python plan builder and the CUDA plan
(`csrc/sipg_plan.h`).  `tests/test_capi.py` checks both sides agree through
`sipg_abi_layout()` exported by libsipg.so.
"""
import numpy as np

ABI_VERSION = 5

SHAPE_QUAD, SHAPE_TRI, SHAPE_HEX = 0, 1, 2
SHAPE_ID = {"quad": SHAPE_QUAD, "tri": SHAPE_TRI, "hex": SHAPE_HEX}
NFACES = {SHAPE_QUAD: 4, SHAPE_TRI: 3, SHAPE_HEX: 6}
DIM_OF = {SHAPE_QUAD: 2, SHAPE_TRI: 2, SHAPE_HEX: 3}

# --- class descriptor: int32[CD_WORDS] ------------------------------------
CD_WORDS = 64
CD_SHAPE, CD_N, CD_Q0, CD_Q1, CD_Q2, CD_NC, CD_NPHYS, CD_NFACES = range(8)
CD_GEOM, CD_COUNT, CD_ELEM_OFF, CD_REC_OFF, CD_EGEO_OFF, CD_EGEO_STRIDE, CD_GLLMASK, CD_KIND = range(8, 16)
CD_ROLE = 63        # launch role: 0 first, 1 after the halo exchange, 2 ghost (never launched)
# tensor shapes: per axis a, base CD_TAX + 8 a
CD_TAX = 16
TX_V, TX_DV, TX_D, TX_W, TX_VEND, TX_DVEND, TX_LEND, TX_PTS = range(8)
# triangles
CD_TRI = 16
(TR_A, TR_DA, TR_D0, TR_D1, TR_W0, TR_W1, TR_B, TR_DB, TR_GID, TR_AEND, TR_DAEND,
 TR_BM1, TR_DBM1, TR_L0, TR_L1, TR_REFW, TR_PTS0, TR_PTS1, TR_GSTART) = range(16, 35)

GEOM_REGULAR, GEOM_POINTWISE = 0, 1

# --- face record (128 bytes) ----------------------------------------------
FT_BOUNDARY, FT_DIRECT, FT_SHARED = 0, 1, 2
F_SELF_PW = 1       # self swj / Gn pointwise (pool block at geo)
F_OTHER_PW = 2      # other Gn pointwise (direct: nbr_rec block; shared: own block)
F_OTHER_ID = 4      # other face grid -> flux grid is the identity
F_OTHER_SWAP = 8    # flux axis k <- other axis 1-k
F_SELF_ID = 16      # own face grid -> flux grid is the identity
F_SELF_SWAP = 32
F_SELF_NEG = 64     # triangle chain: self face parameter at flux point = -t
F_OTHER_NEG = 128
F_FAST_HEX = 256    # conforming same-class hex neighbour, identity grid, constant metric,
                    # normal-only neighbour metric: register-column fast path
F_FAST_SHARED = 512  # hex shared trace, no axis swap, constant metric, normal-only metrics:
                     # neighbour planes evaluated at the trace grid with 1-D tables (k_hexp)

FACE_REC = np.dtype([
    ("type", "<i4"), ("flags", "<i4"), ("nbr", "<i4"), ("nbr_face", "<i4"),
    ("nbr_rec", "<i4"), ("nt0", "<i4"), ("nt1", "<i4"), ("to0", "<i4"),
    ("to1", "<i4"), ("ts0", "<i4"), ("ts1", "<i4"), ("wt0", "<i4"),
    ("wt1", "<i4"), ("geo", "<i4"), ("nbr_dof", "<i8"),
    ("tau", "<f8"), ("sJ", "<f8"), ("gs", "<f8", (3,)), ("go", "<f8", (3,)),
])
assert FACE_REC.itemsize == 128
