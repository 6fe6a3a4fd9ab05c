/*
 * ORACLE / TEST INFRASTRUCTURE ONLY — a CPU restatement, in plain C, of the
 * reference deltaflux engine path (/root/reference/proj/src/{engine,
 * delta_layers, buffer_manager, alignment, tile_grid, network}.cpp).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load it, and only as the checker. The product (paper_2210_09887_b200) never
 * links or calls it.
 *
 * Parity pinned: tests/test_oracle.py checks this restatement bit-for-bit
 * against (a) the unmodified reference built by oracle/Makefile
 * (oracle/_ref/libdfxref.so) on random networks / sequences, and (b) the
 * committed golden fixtures in tests/golden/ that tests/golden/make_golden.py
 * generated from that reference build.
 *
 * API: the same entry points as include/dfx_b200.h with the dfo_ prefix.
 */
#ifndef DFX_ORACLE_H
#define DFX_ORACLE_H

#include "dfx_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct dfo_engine dfo_engine;

const char* dfo_last_error(void);
int dfo_create(const dfx_net_desc* net, const dfx_engine_config* cfg, dfo_engine** out);
void dfo_destroy(dfo_engine* e);
int dfo_run_frame(dfo_engine* e, const float* frame, int c, int h, int w, const float* h9,
                  const float* roi, dfx_frame_info* info, float* out, size_t out_cap);
int dfo_reset(dfo_engine* e);
int dfo_input_mask(dfo_engine* e, uint8_t* out, size_t cap, int* th, int* tw);
int dfo_layer_flops(dfo_engine* e, const char* name, uint64_t* flops, uint64_t* dense);
int dfo_grid(dfo_engine* e, int* rows, int* cols);
int dfo_read_state(dfo_engine* e, const char* layer, int which, float* out, size_t cap, int* c,
                   int* h, int* w);
int dfo_read_packet(dfo_engine* e, const char* layer, float* out, size_t cap, int* c, int* gh,
                    int* gw, int* halo, uint8_t* mask, size_t mask_cap);
int dfo_read_ledger(dfo_engine* e, int* used, int64_t* ty, int64_t* tx, uint8_t* covered,
                    size_t cap);
/* Network facts from the restated validate() (network.cpp:46-254):
 * ring width, and per layer: kind, in/out channels, in/out tile, halo in/out. */
int dfo_net_info(dfo_engine* e, int* ring, int* num_layers);
int dfo_layer_info(dfo_engine* e, int layer, int* info7, float* beta, size_t beta_cap);

#ifdef __cplusplus
}
#endif
#endif
