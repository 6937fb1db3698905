// Device-side batch planning (devplan.cu): layouts shared with pjg_api.cu.
#pragma once

#include "../../include/pjg.h"
#include "pjg_internal.h"

namespace pjg {

// parse() result of one file (header only; offsets are file-relative)
struct DevHdr {
    int32_t status, table_status;
    uint32_t width, height, ncomp, h_max, v_max, mcus_x, mcus_y, dpm;
    uint32_t restart_interval, pad;
    uint64_t scan_start;
    uint64_t du_comp, du_kslot;
    uint8_t cid[3], ch[3], cv[3], tq[3], td[3], ta[3];
    uint8_t q_present, dc_present, ac_present, pad2;
    uint8_t q_prec[4];
    uint64_t q_off[4], dc_off[4], ac_off[4];  // DQT values / DHT counts
    uint16_t dc_n[4], ac_n[4];                 // DHT symbol counts
    uint16_t dc_id[3], ac_id[3], q_id[3];      // batch-unique table ids (P2)
    uint16_t pad3;
};

// representative of a unique table: absolute offset in the raw buffer
struct TabRep {
    uint64_t off;
    uint32_t nsym;
    uint32_t kind;  // 0 DC, 1 AC, 2 quantiser
    uint32_t prec;
    uint32_t pad;
};

struct PlanTotals {
    uint64_t sub, du, outb, seg, bits, raw, n_ok, max_du;
    uint32_t k0t, k4t, ndri, all420, n_huff, n_quant;
};

// per-image layout counts (the host planner's pass-1 counts)
struct Cnt {
    unsigned long long sub, du, outb, seg;
    uint32_t k0t, k4t, ndri, pad;
};

enum PlanCounter { kPlanHuff = 0, kPlanQuant = 1, kPlanCounters = 4 };

struct PlanParams {
    const uint8_t* raw;        // the uploaded files
    const uint64_t* offsets;   // file i at raw + offsets[i]
    const uint64_t* sizes;
    uint32_t n;
    uint32_t allow_dri;
    uint32_t out_mode;
    uint32_t k0_bpt;
    uint64_t sb_int;
    DevHdr* hdr;
    // dedup
    uint64_t* hkeys;
    uint32_t* hval;
    TabRep* hrep;
    uint32_t hmask;
    uint32_t* counters;
    TabRep* uh;                // unique Huffman tables (by id)
    TabRep* uq;                // unique quantisers
    // layout outputs
    ImgDesc* desc;
    ImgState* state;
    ImgState* state0;          // initial statuses (decode re-runs start from them)
    pjg_image_info* info;
    uint32_t* k0_first;
    uint32_t* tile_first;
    uint64_t* sub_first;
    uint32_t* dri;
    PlanTotals* totals;
    Cnt* cnt;                  // per image
    Cnt* blk;                  // per layout CTA: totals, then exclusive prefixes
};

struct TableOut {
    DevHuff* huff;
    uint16_t* quant;  // column-major, 64 per table
    float* wq;
    uint32_t n_huff, n_quant;
};

void launch_plan_parse(const PlanParams& p, void* stream);
void launch_plan_finish(const PlanParams& p, const TableOut& t, uint32_t* k0img, uint32_t* subimg,
                        uint64_t n_subimg, void* stream);

}  // namespace pjg
