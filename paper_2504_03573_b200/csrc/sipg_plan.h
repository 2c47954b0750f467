// Device plan layout shared with paper_2504_03573_b200/layout.py.
// Any change here must bump SIPG_ABI_VERSION and layout.ABI_VERSION.
#pragma once
#include <stdint.h>

#define SIPG_ABI_VERSION 5

enum { SHAPE_QUAD = 0, SHAPE_TRI = 1, SHAPE_HEX = 2 };
enum { GEOM_REGULAR = 0, GEOM_POINTWISE = 1 };

// class descriptor words (int32[CD_WORDS])
#define CD_WORDS 64
enum {
  CD_SHAPE = 0, CD_N, CD_Q0, CD_Q1, CD_Q2, CD_NC, CD_NPHYS, CD_NFACES,
  CD_GEOM, CD_COUNT, CD_ELEM_OFF, CD_REC_OFF, CD_EGEO_OFF, CD_EGEO_STRIDE, CD_GLLMASK, CD_KIND,
  CD_TAX = 16,
  CD_ROLE = 63   // launch role: 0 first, 1 after the halo exchange, 2 ghost (never launched)
};
enum { TX_V = 0, TX_DV, TX_D, TX_W, TX_VEND, TX_DVEND, TX_LEND, TX_PTS };
enum {
  TR_A = 16, TR_DA, TR_D0, TR_D1, TR_W0, TR_W1, TR_B, TR_DB, TR_GID, TR_AEND, TR_DAEND,
  TR_BM1, TR_DBM1, TR_L0, TR_L1, TR_REFW, TR_PTS0, TR_PTS1, TR_GSTART
};

enum { FT_BOUNDARY = 0, FT_DIRECT = 1, FT_SHARED = 2 };
enum {
  F_SELF_PW = 1, F_OTHER_PW = 2, F_OTHER_ID = 4, F_OTHER_SWAP = 8,
  F_SELF_ID = 16, F_SELF_SWAP = 32, F_SELF_NEG = 64, F_OTHER_NEG = 128,
  F_FAST_HEX = 256,  // conforming same-class hex neighbour, identity grid, constant metric, normal-only
  F_FAST_SHARED = 512  // hex shared trace, no swap, constant metric, normal-only: planes + 1-D tables
};

struct FaceRec {            // 128 bytes, numpy dtype layout.FACE_REC
  int32_t type, flags, nbr, nbr_face, nbr_rec, nt0, nt1, to0, to1, ts0, ts1, wt0, wt1, geo;
  int64_t nbr_dof;          // dof offset of the neighbour (-1 on boundary faces)
  double tau, sJ, gs[3], go[3];
};
static_assert(sizeof(FaceRec) == 128, "FaceRec layout");

struct DevPlan {
  const int32_t* cd;           // n_cls * CD_WORDS
  const int32_t* class_elems;  // per class, element ids
  const int32_t* elem_class;   // per element
  const int32_t* elem_pos;     // per element: index within its class
  const int64_t* dof_off;      // per element (+1)
  const FaceRec* recs;         // per class: count * nfaces, class-contiguous
  const double* tab;           // table pool
  const double* egeo;          // element geometry pool
  const double* fgeo;          // face pointwise geometry pool
  double lam;
  int32_t dim;
  int32_t n_cls;
  int32_t debug;               // instrumentation bits (SIPG_DEBUG env): 1 = skip face work (timing only)
  int32_t pad;
  double* planes;              // published face planes (hex): per element 6 faces x (u-plane, dn-plane)
  const int64_t* plane_off;    // per element offset into planes (-1: none)
  const int64_t* rec_ext;      // per face record, 2 words: [0] nbr face planes offset | N_o << 48,
                               //                           [1] E_o axis-0 table | axis-1 table << 32
};
