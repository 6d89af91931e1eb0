// occx_host.cpp -- native host side of ScorePlan / score_space() (CPython
// extension module paper_1701_08547_b200._occx_host).
//
// The scorer's e2e step is: host space description -> one H2D blob -> K1 +
// feature table + K2i + K3 on the GPU -> D2H top-k -> decoded configurations.
// The two host ends are per-object Python work (tuples of dimension values,
// InstructionMix dicts, Ranked entries); this module does them in C++:
//
//   pack_plan(dims, var_counts, mixes, tstars, device_id, DeviceError)
//       -> (blob: bytearray, offsets: 5-tuple, total, n_pool, seg_start list)
//     the same bytes ScorePlan.__init__ built with numpy (include/occx.h
//     occx_segdesc_t rows | u32 value pool | u64 masks[n_seg][3] | u32
//     var_kernel | occx_mix_t rows, each part 256-byte aligned), with the
//     same validation and messages:
//       * TC/BC/REGS/SMEM values: non-negative ints (anything with
//         __index__), clamped to 2^32-1 in the pool;
//       * membership masks = tuning.membership_masks (ref tuning.py:94-127):
//         kept = [t in TC if t in T*] in space order (duplicates counted),
//         sorted, ceil-half lower / upper, bit t/32 - 1;
//       * mixes = batch.pack_mixes: counts by device class id, first_key =
//         dict insertion rank (ref mix.py:245-261 order), counts above
//         2^32-1 raise DeviceError.
//   decode(keys, n_arch, k, total, seg_start, kern_dims, var_base)
//       -> list (per segment) of lists of Ranked
//     = ScorePlan.decode's per-entry unpacking (key bits, global index ->
//     enumerate_space digits, last dimension fastest, ref tuning.py:70-77),
//     Ranked being a C struct sequence (no Python __init__ per entry).
#define PY_SSIZE_T_CLEAN
#include <Python.h>
#include <structmember.h>

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <vector>

namespace {

constexpr uint64_t kU32Max = 0xffffffffull;
constexpr uint64_t kIdxMask = (1ull << 34) - 1;
constexpr size_t kSegDescBytes = 80, kMixBytes = 144;

size_t align256(size_t n) { return (std::max<size_t>(n, 1) + 255) / 256 * 256; }

// A non-negative Python integer (or __index__ object) -> value clamped to
// 2^32-1; false (ValueError set) otherwise.  Mirrors batch._nonneg_ints.
bool nonneg_u32(PyObject* v, uint32_t* out) {
  if (PyFloat_Check(v) || PyUnicode_Check(v) || PyBytes_Check(v)) goto bad;
  {
    PyObject* i = PyNumber_Index(v);
    if (!i) {
      PyErr_Clear();
      goto bad;
    }
    int overflow = 0;
    const long long x = PyLong_AsLongLongAndOverflow(i, &overflow);
    Py_DECREF(i);
    if (overflow < 0 || (overflow == 0 && x < 0)) goto bad;
    if (overflow == 0 && x == -1 && PyErr_Occurred()) return false;
    *out = (overflow > 0 || (uint64_t)x > kU32Max) ? (uint32_t)kU32Max : (uint32_t)x;
    return true;
  }
bad:
  PyErr_SetString(PyExc_ValueError, "TC/BC/REGS/SMEM values must be non-negative ints");
  return false;
}

// Mask bit of a thread count: t/32 - 1 for t % 32 == 0, 32 <= t <= 2048; -1
// for values no mask can hold (they cannot be in T* of an accepted arch).
int mask_bit(PyObject* v) {
  int overflow = 0;
  long long t = -1;
  if (PyLong_Check(v)) {
    t = PyLong_AsLongLongAndOverflow(v, &overflow);
  } else if (!PyFloat_Check(v)) {           // numpy integers compare equal to ints
    PyObject* i = PyNumber_Index(v);
    if (i) {
      t = PyLong_AsLongLongAndOverflow(i, &overflow);
      Py_DECREF(i);
    }
  }
  PyErr_Clear();
  if (overflow || t < 32 || t > 2048 || (t & 31)) return -1;
  return (int)(t >> 5) - 1;
}

struct Masks {
  uint64_t st, lo, hi;
};

// tuning.membership_masks for one (TC, T*) pair; T* given as its bitset.
// A thread count that equals a T* member but lies outside the bitset
// cannot occur (T* <= max_threads_per_block <= 2048, arch.device_limits_ok).
Masks masks_of(PyObject* tc_fast, uint64_t tstar) {
  int cnt[64] = {0};
  Py_ssize_t n = PySequence_Fast_GET_SIZE(tc_fast);
  PyObject** it = PySequence_Fast_ITEMS(tc_fast);
  int kept = 0;
  for (Py_ssize_t i = 0; i < n; ++i) {
    const int b = mask_bit(it[i]);
    if (b >= 0 && ((tstar >> b) & 1u)) {
      ++cnt[b];
      ++kept;
    }
  }
  Masks m{0, 0, 0};
  if (kept == 0) return m;                       // NoCandidatesError: no member bits
  const int h = kept - kept / 2;                 // ceil half (ref tuning.py:118-120)
  int seen = 0;
  for (int b = 0; b < 64; ++b) {
    if (!cnt[b]) continue;
    m.st |= 1ull << b;
    if (seen < h) m.lo |= 1ull << b;             // some of the h smallest
    if (seen + cnt[b] > kept - h) m.hi |= 1ull << b;   // some of the h largest
    seen += cnt[b];
  }
  return m;
}

PyObject* pack_plan(PyObject*, PyObject* args) {
  PyObject *dims, *var_counts, *mixes, *tstars, *device_id, *dev_err;
  if (!PyArg_ParseTuple(args, "OOOOOO", &dims, &var_counts, &mixes, &tstars, &device_id,
                        &dev_err))
    return nullptr;
  PyObject* dims_f = PySequence_Fast(dims, "dims must be a sequence");
  if (!dims_f) return nullptr;
  PyObject* ts_f = PySequence_Fast(tstars, "tstars must be a sequence");
  PyObject* vc_f = ts_f ? PySequence_Fast(var_counts, "var_counts must be a sequence") : nullptr;
  PyObject* mx_f = vc_f ? PySequence_Fast(mixes, "mixes must be a sequence") : nullptr;
  std::vector<PyObject*> owned{dims_f, ts_f, vc_f, mx_f};
  auto fail = [&]() -> PyObject* {
    for (PyObject* o : owned) Py_XDECREF(o);
    return nullptr;
  };
  if (!mx_f) return fail();
  const Py_ssize_t n_kern = PySequence_Fast_GET_SIZE(dims_f);
  const Py_ssize_t n_arch = PySequence_Fast_GET_SIZE(ts_f);
  const Py_ssize_t n_mix = PySequence_Fast_GET_SIZE(mx_f);
  if (PySequence_Fast_GET_SIZE(vc_f) != n_kern) {
    PyErr_SetString(PyExc_ValueError, "var_counts length");
    return fail();
  }
  // T* bitsets per arch
  std::vector<uint64_t> tbits(n_arch, 0);
  for (Py_ssize_t a = 0; a < n_arch; ++a) {
    PyObject* f = PySequence_Fast(PySequence_Fast_GET_ITEM(ts_f, a), "T* must be a sequence");
    if (!f) return fail();
    for (Py_ssize_t i = 0; i < PySequence_Fast_GET_SIZE(f); ++i) {
      const int b = mask_bit(PySequence_Fast_GET_ITEM(f, i));
      if (b >= 0) tbits[a] |= 1ull << b;
    }
    Py_DECREF(f);
  }
  const size_t n_seg = (size_t)n_kern * (size_t)n_arch;
  std::vector<uint64_t> seg_desc_words(n_seg * (kSegDescBytes / 8), 0);
  std::vector<uint32_t> pool;
  std::vector<uint64_t> masks(n_seg * 3, 0);
  std::vector<uint32_t> var_kernel;
  uint64_t start = 0;
  uint32_t var_base = 0;
  for (Py_ssize_t ki = 0; ki < n_kern; ++ki) {
    PyObject* kd = PySequence_Fast(PySequence_Fast_GET_ITEM(dims_f, ki), "kernel dims");
    if (!kd) return fail();
    owned.push_back(kd);
    if (PySequence_Fast_GET_SIZE(kd) != 7) {
      PyErr_SetString(PyExc_ValueError, "seven dimensions per kernel");
      return fail();
    }
    uint32_t off[7], len[7];
    uint64_t size = 1;
    PyObject* tc_fast = nullptr;
    for (int j = 0; j < 7; ++j) {
      PyObject* f = PySequence_Fast(PySequence_Fast_GET_ITEM(kd, j), "dimension");
      if (!f) return fail();
      owned.push_back(f);
      const Py_ssize_t m = PySequence_Fast_GET_SIZE(f);
      off[j] = (uint32_t)pool.size();
      len[j] = (uint32_t)m;
      size *= (uint64_t)m;
      PyObject** it = PySequence_Fast_ITEMS(f);
      if (j == 0 || j == 1 || j == 5 || j == 6) {    // value dims; UIF/PL/CFLAGS by index
        for (Py_ssize_t i = 0; i < m; ++i) {
          uint32_t v;
          if (!nonneg_u32(it[i], &v)) return fail();
          pool.push_back(v);
        }
      } else {
        pool.insert(pool.end(), (size_t)m, 0u);
      }
      if (j == 0) tc_fast = f;
    }
    const long nv = PyLong_AsLong(PySequence_Fast_GET_ITEM(vc_f, ki));
    if (nv < 0 && PyErr_Occurred()) return fail();
    // archs sharing T* share the masks
    std::vector<std::pair<uint64_t, Masks>> memo;
    for (Py_ssize_t a = 0; a < n_arch; ++a) {
      const size_t s = (size_t)ki * n_arch + a;
      uint64_t* w = &seg_desc_words[s * (kSegDescBytes / 8)];
      w[0] = start;
      w[1] = size;
      uint32_t* u = reinterpret_cast<uint32_t*>(w + 2);
      u[0] = (uint32_t)a;
      u[1] = var_base;
      std::memcpy(u + 2, off, sizeof(off));
      std::memcpy(u + 9, len, sizeof(len));
      start += size;
      Masks mk;
      auto hit = std::find_if(memo.begin(), memo.end(),
                              [&](const std::pair<uint64_t, Masks>& e) { return e.first == tbits[a]; });
      if (hit != memo.end()) {
        mk = hit->second;
      } else {
        mk = masks_of(tc_fast, tbits[a]);
        memo.emplace_back(tbits[a], mk);
      }
      masks[3 * s] = mk.st;
      masks[3 * s + 1] = mk.lo;
      masks[3 * s + 2] = mk.hi;
    }
    var_kernel.insert(var_kernel.end(), (size_t)nv, (uint32_t)ki);
    var_base += (uint32_t)nv;
  }
  if ((Py_ssize_t)var_kernel.size() != n_mix) {
    PyErr_SetString(PyExc_ValueError, "need one mix per (UIF, CFLAGS) variant");
    return fail();
  }
  if (pool.empty()) pool.push_back(0);
  // blob layout: desc | pool | masks | var_kernel | mixes
  const size_t sizes[5] = {n_seg * kSegDescBytes, pool.size() * 4, masks.size() * 8,
                           var_kernel.size() * 4, (size_t)n_mix * kMixBytes};
  size_t offs[5], total_b = 0;
  for (int i = 0; i < 5; ++i) {
    offs[i] = total_b;
    total_b += align256(sizes[i]);
  }
  PyObject* blob = PyByteArray_FromStringAndSize(nullptr, (Py_ssize_t)total_b);
  if (!blob) return fail();
  owned.push_back(blob);
  char* b = PyByteArray_AS_STRING(blob);
  std::memset(b, 0, total_b);
  std::memcpy(b + offs[0], seg_desc_words.data(), sizes[0]);
  std::memcpy(b + offs[1], pool.data(), sizes[1]);
  std::memcpy(b + offs[2], masks.data(), sizes[2]);
  if (sizes[3]) std::memcpy(b + offs[3], var_kernel.data(), sizes[3]);
  // occx_mix_t: u32 counts[16] | u32 first_key[16] | u64 reg_operands | u32 n_instr | u32 rsv
  for (Py_ssize_t i = 0; i < n_mix; ++i) {
    PyObject* m = PySequence_Fast_GET_ITEM(mx_f, i);
    char* row = b + offs[4] + (size_t)i * kMixBytes;
    uint32_t* counts = reinterpret_cast<uint32_t*>(row);
    uint32_t* first = counts + 16;
    for (int c = 0; c < 16; ++c) first[c] = (uint32_t)kU32Max;
    PyObject* d = PyObject_GetAttrString(m, "counts");
    if (!d) return fail();
    if (!PyDict_Check(d)) {
      Py_DECREF(d);
      PyErr_SetString(PyExc_TypeError, "InstructionMix.counts must be a dict");
      return fail();
    }
    Py_ssize_t pos = 0, rank = 0;
    PyObject *key, *val;
    uint64_t total = 0;
    while (PyDict_Next(d, &pos, &key, &val)) {
      PyObject* id = PyDict_GetItemWithError(device_id, key);
      if (!id) {
        Py_DECREF(d);
        if (!PyErr_Occurred()) PyErr_SetObject(PyExc_KeyError, key);
        return fail();
      }
      const long di = PyLong_AsLong(id);
      int overflow = 0;
      const long long c = PyLong_AsLongLongAndOverflow(val, &overflow);
      if (overflow || c < 0 || (uint64_t)c > kU32Max) {
        Py_DECREF(d);
        PyErr_Clear();
        PyErr_SetString(dev_err, "per-class count above 2^32-1");
        return fail();
      }
      counts[di] = (uint32_t)c;
      first[di] = (uint32_t)rank++;
      total += (uint64_t)c;
    }
    Py_DECREF(d);
    PyObject* r = PyObject_GetAttrString(m, "reg_operands");
    if (!r) return fail();
    const unsigned long long regs = PyLong_AsUnsignedLongLong(r);
    Py_DECREF(r);
    if (regs == (unsigned long long)-1 && PyErr_Occurred()) {
      PyErr_Clear();
      PyErr_SetString(dev_err, "reg_operands above 2^64-1");
      return fail();
    }
    std::memcpy(row + 128, &regs, 8);
    const uint32_t n_instr = (uint32_t)std::min<uint64_t>(total, kU32Max);
    std::memcpy(row + 136, &n_instr, 4);
  }
  PyObject* starts = PyList_New((Py_ssize_t)n_seg);
  if (!starts) return fail();
  owned.push_back(starts);
  for (size_t i = 0; i < n_seg; ++i) {
    PyObject* v = PyLong_FromUnsignedLongLong(seg_desc_words[i * (kSegDescBytes / 8)]);
    if (!v) return fail();
    PyList_SET_ITEM(starts, (Py_ssize_t)i, v);
  }
  PyObject* res = Py_BuildValue("O(nnnnn)KnO", blob, (Py_ssize_t)offs[0], (Py_ssize_t)offs[1],
                                (Py_ssize_t)offs[2], (Py_ssize_t)offs[3], (Py_ssize_t)offs[4],
                                (unsigned long long)start, (Py_ssize_t)pool.size(), starts);
  fail();   // drop our references (blob is held by res)
  return res;
}

// ---- decode -----------------------------------------------------------------
PyTypeObject* RankedType = nullptr;

PyStructSequence_Field kRankedFields[] = {
    {"index", "global candidate index"},
    {"config", "enumerate_space(kernel.space) tuple"},
    {"variant", "variant index (kernel's var_base + UIF index * |CFLAGS| + CFLAGS index)"},
    {"arch", "arch index"},
    {"active_warps", "active warps per SM (key bits 60-54)"},
    {"rule_keep", "survives rule_prune (key bit 62)"},
    {"static_keep", "survives static_prune (key bit 61)"},
    {"cost_rank", "dense cost rank among the kernel's variants, None if unsupported"},
    {"key", "the u64 scoring key"},
    {nullptr, nullptr}};

PyStructSequence_Desc kRankedDesc = {
    "paper_1701_08547_b200.Ranked",
    "One entry of a segment's top-k list, decoded from its key.", kRankedFields, 9};

PyObject* decode(PyObject*, PyObject* args) {
  Py_buffer kb;
  Py_ssize_t n_arch, k;
  unsigned long long total;
  PyObject *seg_start, *kern_dims, *var_base;
  if (!PyArg_ParseTuple(args, "y*nnKOOO", &kb, &n_arch, &k, &total, &seg_start, &kern_dims,
                        &var_base))
    return nullptr;
  PyObject* out = nullptr;
  PyObject *kd_f = nullptr, *ss_f = nullptr, *vb_f = nullptr;
  std::vector<PyObject*> dim_f;
  const uint64_t* keys = static_cast<const uint64_t*>(kb.buf);
  const Py_ssize_t n_kern = PySequence_Size(kern_dims);
  const Py_ssize_t n_seg = n_kern * n_arch;
  if (n_kern < 0 || kb.len < (Py_ssize_t)(n_seg * k * 8) || total == 0) {
    if (!PyErr_Occurred()) PyErr_SetString(PyExc_ValueError, "decode: bad arguments");
    PyBuffer_Release(&kb);
    return nullptr;
  }
  kd_f = PySequence_Fast(kern_dims, "kern_dims");
  if (!kd_f) goto done;
  ss_f = PySequence_Fast(seg_start, "seg_start");
  if (!ss_f) goto done;
  vb_f = PySequence_Fast(var_base, "var_base");
  if (!vb_f) goto done;
  if (PySequence_Fast_GET_SIZE(ss_f) < n_seg || PySequence_Fast_GET_SIZE(vb_f) < n_kern) {
    PyErr_SetString(PyExc_ValueError, "decode: seg_start / var_base too short");
    goto done;
  }
  out = PyList_New(n_seg);
  if (!out) goto done;
  for (Py_ssize_t ki = 0; ki < n_kern; ++ki) {
    PyObject* dims = PySequence_Fast(PySequence_Fast_GET_ITEM(kd_f, ki), "dims");
    if (!dims) goto fail;
    dim_f.push_back(dims);
    const Py_ssize_t nd = PySequence_Fast_GET_SIZE(dims);
    std::vector<PyObject*> cols(nd);
    std::vector<uint64_t> lens(nd);
    for (Py_ssize_t d = 0; d < nd; ++d) {
      PyObject* c = PySequence_Fast(PySequence_Fast_GET_ITEM(dims, d), "dimension");
      if (!c) goto fail;
      dim_f.push_back(c);
      cols[d] = c;
      lens[d] = (uint64_t)PySequence_Fast_GET_SIZE(c);
    }
    const long long vb = PyLong_AsLongLong(PySequence_Fast_GET_ITEM(vb_f, ki));
    if (vb == -1 && PyErr_Occurred()) goto fail;
    const uint64_t n_cf = nd > 4 ? lens[4] : 1;
    for (Py_ssize_t a = 0; a < n_arch; ++a) {
      const Py_ssize_t s = ki * n_arch + a;
      PyObject* st_o = PySequence_Fast_GET_ITEM(ss_f, s);
      const unsigned long long st = PyLong_AsUnsignedLongLong(st_o);
      if (st == (unsigned long long)-1 && PyErr_Occurred()) goto fail;
      PyObject* entries = PyList_New(0);
      if (!entries) goto fail;
      PyList_SET_ITEM(out, s, entries);
      for (Py_ssize_t j = 0; j < k; ++j) {
        const uint64_t key = keys[s * k + j];
        if (key == 0) continue;
        const uint64_t idx = kIdxMask - (key & kIdxMask);
        uint64_t rem = idx % total - st;                 // local index within the segment
        PyObject* cfg = PyTuple_New(nd);
        if (!cfg) goto fail;
        uint64_t dig2 = 0, dig4 = 0;
        for (Py_ssize_t d = nd - 1; d >= 0; --d) {      // last dimension fastest
          const uint64_t r = rem % lens[d];
          rem /= lens[d];
          if (d == 2) dig2 = r;
          if (d == 4) dig4 = r;
          PyObject* v = PySequence_Fast_GET_ITEM(cols[d], (Py_ssize_t)r);
          Py_INCREF(v);
          PyTuple_SET_ITEM(cfg, d, v);
        }
        const uint32_t rbits = (uint32_t)((key >> 34) & 0xFFFFFu);
        PyObject* e = PyStructSequence_New(RankedType);
        if (!e) {
          Py_DECREF(cfg);
          goto fail;
        }
        PyStructSequence_SET_ITEM(e, 0, PyLong_FromUnsignedLongLong(idx));
        PyStructSequence_SET_ITEM(e, 1, cfg);
        PyStructSequence_SET_ITEM(e, 2, PyLong_FromLongLong(vb + (long long)(dig2 * n_cf + dig4)));
        PyStructSequence_SET_ITEM(e, 3, PyLong_FromSsize_t(a));
        PyStructSequence_SET_ITEM(e, 4, PyLong_FromUnsignedLong((unsigned long)((key >> 54) & 0x7F)));
        PyObject* rk = (key >> 62) & 1 ? Py_True : Py_False;
        PyObject* sk = (key >> 61) & 1 ? Py_True : Py_False;
        Py_INCREF(rk);
        Py_INCREF(sk);
        PyStructSequence_SET_ITEM(e, 5, rk);
        PyStructSequence_SET_ITEM(e, 6, sk);
        PyObject* cr;
        if (rbits) {
          cr = PyLong_FromUnsignedLong((1u << 20) - 1u - rbits);
        } else {
          cr = Py_None;
          Py_INCREF(cr);
        }
        PyStructSequence_SET_ITEM(e, 7, cr);
        PyStructSequence_SET_ITEM(e, 8, PyLong_FromUnsignedLongLong(key));
        if (PyErr_Occurred() || PyList_Append(entries, e) < 0) {
          Py_DECREF(e);
          goto fail;
        }
        Py_DECREF(e);
      }
    }
  }
  goto done;
fail:
  Py_CLEAR(out);
done:
  for (PyObject* o : dim_f) Py_DECREF(o);
  Py_XDECREF(kd_f);
  Py_XDECREF(ss_f);
  Py_XDECREF(vb_f);
  PyBuffer_Release(&kb);
  return out;
}

PyMethodDef kMethods[] = {
    {"pack_plan", pack_plan, METH_VARARGS,
     "pack_plan(dims, var_counts, mixes, tstars, device_id, DeviceError) -> "
     "(blob, offsets, total, n_pool, seg_start)"},
    {"decode", decode, METH_VARARGS,
     "decode(keys, n_arch, k, total, seg_start, kern_dims, var_base) -> [[Ranked]]"},
    {nullptr, nullptr, 0, nullptr}};

PyModuleDef kModule = {PyModuleDef_HEAD_INIT, "_occx_host",
                       "Native host side of ScorePlan (packing, decoding).", -1, kMethods};

}  // namespace

PyMODINIT_FUNC PyInit__occx_host(void) {
  PyObject* m = PyModule_Create(&kModule);
  if (!m) return nullptr;
  if (!RankedType) {
    RankedType = PyStructSequence_NewType(&kRankedDesc);
    if (!RankedType) return nullptr;
  }
  Py_INCREF(RankedType);
  if (PyModule_AddObject(m, "Ranked", reinterpret_cast<PyObject*>(RankedType)) < 0) return nullptr;
  return m;
}
