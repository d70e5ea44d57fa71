/* leo_front.h — native listing front-end.
 *
 * Replaces the reference's host front-end for the hot path's inputs:
 *   disasm.parse_listing   (disasm.py:259-409)  listing text -> instructions
 *   disasm.build_cfg       (disasm.py:495-607)  basic blocks, edges, diagnostics
 *   disasm.parse_kernels   (disasm.py:618-626)  one CFG per kernel section
 *   soa.encode_cfg         (the SoA layout of include/leo_b200.h, LeoKernel)
 * in one C++ pass, emitting the structure-of-arrays the device library takes
 * directly (no per-instruction Python objects).  Error behaviour follows the
 * reference: the first ListingError is reported with its exact message text
 * (`message near 'token' (line L, col C)`).
 *
 * Host-only library (libleo_front.so), plain C ABI. */
#ifndef LEO_FRONT_H
#define LEO_FRONT_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* dialect: 0 nvidia, 1 amd, 2 intel.  table_text: the opcode table
 * (`<prefix> <class>` lines, isa.py OpcodeTable.parse format). */
void* leo_front_parse(int32_t dialect, const char* text, int64_t len, const char* table_text,
                      int64_t table_len);
/* 0 on success, else the error message length (copied into buf, NUL-terminated) */
int32_t leo_front_error(void* h, char* buf, int32_t cap);
int32_t leo_front_n_kernels(void* h);
const char* leo_front_kernel_name(void* h, int32_t k);
/* sizes[0..7] = N, B, operand records, succ entries, pred entries, units,
 * line keys, cfg diagnostics */
int32_t leo_front_sizes(void* h, int32_t k, int64_t* sizes);
/* copy kernel k's SoA into caller buffers sized by leo_front_sizes */
int32_t leo_front_arrays(void* h, int32_t k, uint8_t* opclass, int32_t* block_of, int32_t* opnd_ptr,
                         uint32_t* opnd, uint8_t* sync_kind, uint32_t* sync_a, uint32_t* sync_b,
                         int32_t* blk_first, int32_t* blk_last, int32_t* succ_ptr, int32_t* succ,
                         int32_t* pred_ptr, int32_t* pred, int32_t* unit_base, int64_t* offset,
                         int32_t* line_id);
/* strings of kernel k: which 0 mnemonic[i], 1 str(src_loc)[i] (NULL when
 * absent), 2 line key[i], 3 cfg diagnostic[i] */
const char* leo_front_string(void* h, int32_t k, int32_t which, int32_t i);
/* all strings `which` of kernel k joined by '\n' (absent src_loc = empty
 * line) into buf; returns the byte length needed (call with cap 0 to size) */
int64_t leo_front_strings(void* h, int32_t k, int32_t which, char* buf, int64_t cap);
void leo_front_free(void* h);

/* ---- profile documents (native/leo_profile.cpp) ----------------------------
 * Replaces profile.load_profiles (profile.py:244-263, _load_one :186-241, the
 * InstructionSamples / KernelProfile invariants :124-165) and profile.attach
 * (:332-366) + soa.encode_profile.  The JSON document is decoded with CPython
 * json.JSONDecoder.raw_decode semantics; the first error is reported with the
 * reference's exact message text. */
void* leo_profile_parse(const char* text, int64_t len);
/* 0 ok, 1 ProfileError, 2 InputError (unknown vendor), 3 value outside the
 * SoA's integer range; message copied into buf (NUL-terminated), its length
 * in *len */
int32_t leo_profile_error(void* h, char* buf, int32_t cap, int32_t* len);
int32_t leo_profile_n_kernels(void* h);
const char* leo_profile_kernel_name(void* h, int32_t k);
/* info[0..2] = dialect, sampling period (cycles), record count */
int32_t leo_profile_info(void* h, int32_t k, int64_t* info);
/* records in document order; total / exec -1 = absent; cls [n, 8] counts per
 * CommonStall (profile.py:29-43 order) */
int32_t leo_profile_records(void* h, int32_t k, int64_t* offset, int64_t* lat, int64_t* total,
                            int64_t* exec, double* eff, int64_t* cls);
/* attach kernel k to a CFG (name, dialect, n instruction offsets): fills the
 * LeoProfile columns lat i32[n], cls_cnt i32[n*8], exec i64[n], total i32[n],
 * eff f64[n], sampled u8[n]; 0 or the error kind (leo_profile_error) */
int32_t leo_profile_attach(void* h, int32_t k, const char* cfg_name, int32_t cfg_dialect, int32_t n,
                           const int64_t* instr_offset, int32_t* lat, int32_t* cls, int64_t* exec,
                           int32_t* total, double* eff, uint8_t* sampled);
/* the skid diagnostic of the last attach ("" when every offset matched) */
const char* leo_profile_diagnostic(void* h);
void leo_profile_free(void* h);

#ifdef __cplusplus
}
#endif
#endif
