// Non-GEMM kernels of the prompt() hot path (declarations + parameter blocks).
#pragma once
#include <cstdint>
#include <cuda.h>
#include "dtype.hpp"

namespace iolmk {

// One attention work item: `nq` consecutive query tokens of one sequence slot, at positions
// pos0 .. pos0+nq-1, whose q rows are m0 .. m0+nq-1 of the step's q buffer. Keys are positions
// 0 .. pos0+nq-1 of the slot (causal), read through the slot's page table.
struct AttnGroup {
  int slot;
  int m0;
  int nq;
  int pos0;
};

struct AttnParams {
  CUtensorMap q_map;   // prefill: q buffer [T x ldq] as [CB-wide swizzled boxes x 64 rows]
  CUtensorMap kv_map;  // prefill: layer pool as rows of hd ([page][K|V][heads][PAGE] rows), 16-row boxes
  CUtensorMap kvg_map; // decode: the same rows in boxes of decode_heads_per_cta(heads, hd) * PAGE rows
  const h16* q;  // [T x ldq] (head h at columns h*hd ..)
  int ldq;
  h16* z;  // [T x ldz] output
  int ldz;
  const h16* kv;  // layer pool: [page][K|V][heads][PAGE][hd]
  const int* page_table;    // [slots x max_pages]
  int max_pages;
  int heads;
  const AttnGroup* groups;
  int n_groups;
  const uint8_t* key_mask;  // optional: per position validity for slot of forward(); NULL = all valid
  float scale_log2;         // log2(e) / sqrt(hd)
};

}  // namespace iolmk
