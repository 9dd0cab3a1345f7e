// formats.cpp -- the reference's model and trace artefacts on the engine side
// (SURVEY §8f f4), so a C/C++ host runs tree-switched BFS from files with no
// Python in the loop:
//   ADBT model  tree.py:389-447   (serialize / deserialize, byte-identical)
//   trace CSV   adaptive.py:225-254 (write_trace / read_trace, byte-identical:
//               Python's csv module writes "\r\n" line ends)
// ADGR graph files live in graph.cu (they stream into HBM).
// Host-only code: no CUDA here.

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/abfs.h"

namespace abfs {
void set_error(const std::string &msg);
}

namespace {

int fail(int code, const std::string &msg) {
    abfs::set_error(msg);
    return code;
}

// FEATURE_NAMES (features.py:25-35), canonical order.
const char *const kFeatureNames[ABFS_N_FEATURES] = {
    "vertex_count",   "edge_count",     "frontier_abs",  "frontier_pct",    "discovered_abs",
    "discovered_pct", "out_deg.min",    "out_deg.q1",    "out_deg.median",  "out_deg.q3",
    "out_deg.max",    "out_deg.stddev", "in_deg.min",    "in_deg.q1",       "in_deg.median",
    "in_deg.q3",      "in_deg.max",     "in_deg.stddev", "abs_deg.min",     "abs_deg.q1",
    "abs_deg.median", "abs_deg.q3",     "abs_deg.max",   "abs_deg.stddev"};

// KernelId / CountVariant names (kernels.py:40-55) as written in traces.
const char *const kKernelNames[5] = {"EDGE_LIST", "REV_EDGE_LIST", "VERTEX_PUSH", "VERTEX_PULL",
                                     "VERTEX_PUSH_WARP"};
const char *const kVariantNames[3] = {"DIRECT_ATOMIC", "GROUP_REDUCE", "TWO_LEVEL_REDUCE"};

std::string repr_bytes(const unsigned char *b, size_t n) {   // Python repr(bytes)
    bool sq = false, dq = false;
    for (size_t i = 0; i < n; ++i) {
        sq |= b[i] == '\'';
        dq |= b[i] == '"';
    }
    const char q = (sq && !dq) ? '"' : '\'';
    static const char *hex = "0123456789abcdef";
    std::string s = "b";
    s += q;
    for (size_t i = 0; i < n; ++i) {
        const unsigned char c = b[i];
        if (c == (unsigned char)q || c == '\\') {
            s += '\\';
            s += (char)c;
        } else if (c == '\t') {
            s += "\\t";
        } else if (c == '\n') {
            s += "\\n";
        } else if (c == '\r') {
            s += "\\r";
        } else if (c < 0x20 || c >= 0x7f) {
            s += "\\x";
            s += hex[c >> 4];
            s += hex[c & 15];
        } else {
            s += (char)c;
        }
    }
    return s + q;
}

struct File {
    FILE *f = nullptr;
    explicit File(FILE *x) : f(x) {}
    ~File() {
        if (f) fclose(f);
    }
};

}  // namespace

// The owned arrays behind an abfs_tree read from an ADBT file.
struct abfs_tree_file {
    abfs_tree view;
    std::vector<std::string> names;
    std::vector<uint16_t> selection, features;
    std::vector<double> thresholds;
    std::vector<uint32_t> lefts, rights;
    std::vector<uint8_t> classes;
};

extern "C" int abfs_tree_read(const char *path, abfs_tree_file **out) {
    // deserialize (tree.py:409-447): same checks, same messages; the
    // selection names are resolved to canonical feature indices
    // (validate_selection, features.py:53-63).
    if (!path || !out) return fail(ABFS_EINVAL, "null argument");
    File fh(fopen(path, "rb"));
    if (!fh.f) return fail(ABFS_EINVAL, std::string("cannot open model file ") + path);
    unsigned char magic[4];
    const size_t got = fread(magic, 1, 4, fh.f);
    if (got != 4 || std::memcmp(magic, "ADBT", 4) != 0)
        return fail(ABFS_EINVAL, "bad magic " + repr_bytes(magic, got) + " in model file " + path);
    unsigned char hdr[8];
    if (fread(hdr, 1, 8, fh.f) != 8) return fail(ABFS_EINVAL, std::string("truncated model header in ") + path);
    uint32_t version, nodes;
    std::memcpy(&version, hdr, 4);
    std::memcpy(&nodes, hdr + 4, 4);
    if (version != 1) return fail(ABFS_EINVAL, "unsupported model format version " + std::to_string(version));
    uint16_t n_names = 0;
    if (fread(&n_names, 1, 2, fh.f) != 2) return fail(ABFS_EINVAL, std::string("truncated selection header in ") + path);
    abfs_tree_file *t = new abfs_tree_file();
    auto bad = [&](int code, const std::string &m) {
        delete t;
        return fail(code, m);
    };
    for (uint16_t i = 0; i < n_names; ++i) {
        uint16_t len = 0;
        if (fread(&len, 1, 2, fh.f) != 2) return bad(ABFS_EINVAL, std::string("truncated selection name in ") + path);
        std::string nm(len, '\0');
        if (len && fread(&nm[0], 1, len, fh.f) != len)
            return bad(ABFS_EINVAL, std::string("truncated selection name in ") + path);
        t->names.push_back(nm);
    }
    std::vector<unsigned char> body((size_t)nodes * 19);
    if (nodes && fread(body.data(), 1, body.size(), fh.f) != body.size())
        return bad(ABFS_EINVAL, std::string("truncated node records in ") + path);
    if (fgetc(fh.f) != EOF) return bad(ABFS_EINVAL, std::string("trailing bytes in model file ") + path);
    // selection -> canonical indices
    if (t->names.empty()) return bad(ABFS_EINVAL, "feature selection must be non-empty");
    std::string unknown;
    for (size_t i = 0; i < t->names.size(); ++i) {
        for (size_t j = 0; j < i; ++j)
            if (t->names[j] == t->names[i]) return bad(ABFS_EINVAL, "feature selection has duplicate names");
        int idx = -1;
        for (int k = 0; k < ABFS_N_FEATURES; ++k)
            if (t->names[i] == kFeatureNames[k]) idx = k;
        if (idx < 0) unknown += (unknown.empty() ? "'" : ", '") + t->names[i] + "'";
        t->selection.push_back((uint16_t)(idx < 0 ? 0 : idx));
    }
    if (!unknown.empty()) return bad(ABFS_EINVAL, "unknown feature names: [" + unknown + "]");
    // 19-byte packed records <u2 feature, <f8 threshold, <u4 left, <u4 right, u1 class
    t->features.resize(nodes);
    t->thresholds.resize(nodes);
    t->lefts.resize(nodes);
    t->rights.resize(nodes);
    t->classes.resize(nodes);
    for (uint32_t k = 0; k < nodes; ++k) {
        const unsigned char *r = body.data() + (size_t)k * 19;
        std::memcpy(&t->features[k], r, 2);
        std::memcpy(&t->thresholds[k], r + 2, 8);
        std::memcpy(&t->lefts[k], r + 10, 4);
        std::memcpy(&t->rights[k], r + 14, 4);
        t->classes[k] = r[18];
    }
    t->view.node_count = nodes;
    t->view.n_selection = (uint32_t)t->selection.size();
    t->view.selection = t->selection.data();
    t->view.features = t->features.data();
    t->view.thresholds = t->thresholds.data();
    t->view.lefts = t->lefts.data();
    t->view.rights = t->rights.data();
    t->view.leaf_classes = t->classes.data();
    *out = t;
    return ABFS_OK;
}

extern "C" const abfs_tree *abfs_tree_file_view(const abfs_tree_file *t) {
    return t ? &t->view : nullptr;
}

extern "C" void abfs_tree_file_free(abfs_tree_file *t) { delete t; }

extern "C" int abfs_tree_write(const abfs_tree *t, const char *path) {
    // serialize (tree.py:389-406): the selection is written as the canonical
    // feature names of t->selection.
    if (!t || !path) return fail(ABFS_EINVAL, "null argument");
    for (uint32_t i = 0; i < t->n_selection; ++i)
        if (t->selection[i] >= ABFS_N_FEATURES) return fail(ABFS_EINVAL, "bad selection index");
    File fh(fopen(path, "wb"));
    if (!fh.f) return fail(ABFS_EINVAL, std::string("cannot create model file ") + path);
    std::string out = "ADBT";
    auto put = [&](const void *p, size_t n) { out.append(reinterpret_cast<const char *>(p), n); };
    const uint32_t version = 1;
    put(&version, 4);
    put(&t->node_count, 4);
    const uint16_t ns = (uint16_t)t->n_selection;
    put(&ns, 2);
    for (uint32_t i = 0; i < t->n_selection; ++i) {
        const char *nm = kFeatureNames[t->selection[i]];
        const uint16_t len = (uint16_t)std::strlen(nm);
        put(&len, 2);
        put(nm, len);
    }
    for (uint32_t k = 0; k < t->node_count; ++k) {
        put(&t->features[k], 2);
        put(&t->thresholds[k], 8);
        put(&t->lefts[k], 4);
        put(&t->rights[k], 4);
        put(&t->leaf_classes[k], 1);
    }
    if (fwrite(out.data(), 1, out.size(), fh.f) != out.size())
        return fail(ABFS_EINVAL, std::string("write failed: ") + path);
    return ABFS_OK;
}

extern "C" int abfs_trace_write(const char *path, const abfs_level_record *recs, size_t n) {
    // write_trace (adaptive.py:225-234): csv.writer rows, "\r\n" line ends.
    if (!path || (n && !recs)) return fail(ABFS_EINVAL, "null argument");
    File fh(fopen(path, "wb"));
    if (!fh.f) return fail(ABFS_EINVAL, std::string("cannot create trace file ") + path);
    std::string out = "level,kernel,variant,fallback,frontier,elapsed_ns,predict_ns\r\n";
    char line[256];
    for (size_t i = 0; i < n; ++i) {
        const abfs_level_record &r = recs[i];
        if (r.kernel < 0 || r.kernel > 4 || r.variant < 0 || r.variant > 2)
            return fail(ABFS_EINVAL, "bad kernel/variant in record " + std::to_string(i));
        snprintf(line, sizeof line, "%lld,%s,%s,%d,%llu,%llu,%llu\r\n", (long long)r.level,
                 kKernelNames[r.kernel], kVariantNames[r.variant], r.fallback ? 1 : 0,
                 (unsigned long long)r.frontier_size, (unsigned long long)r.elapsed_ns,
                 (unsigned long long)r.prediction_ns);
        out += line;
    }
    if (fwrite(out.data(), 1, out.size(), fh.f) != out.size())
        return fail(ABFS_EINVAL, std::string("write failed: ") + path);
    return ABFS_OK;
}

extern "C" int abfs_trace_read(const char *path, abfs_level_record *recs, size_t cap, size_t *n) {
    // read_trace (adaptive.py:237-254): header must match exactly; the
    // kernel / variant columns are enum names.  new_count / converted are
    // not part of the CSV and come back as 0.
    if (!path || !n) return fail(ABFS_EINVAL, "null argument");
    File fh(fopen(path, "rb"));
    if (!fh.f) return fail(ABFS_EINVAL, std::string("cannot open trace file ") + path);
    std::string text;
    char buf[1 << 16];
    size_t k;
    while ((k = fread(buf, 1, sizeof buf, fh.f)) > 0) text.append(buf, k);
    std::vector<std::string> lines;
    size_t pos = 0;
    while (pos < text.size()) {
        size_t e = text.find('\n', pos);
        if (e == std::string::npos) e = text.size();
        std::string ln = text.substr(pos, e - pos);
        if (!ln.empty() && ln.back() == '\r') ln.pop_back();
        lines.push_back(ln);
        pos = e + 1;
    }
    if (lines.empty() || lines[0] != "level,kernel,variant,fallback,frontier,elapsed_ns,predict_ns")
        return fail(ABFS_EINVAL, std::string("unexpected trace header in ") + path);
    size_t cnt = 0;
    for (size_t i = 1; i < lines.size(); ++i) {
        if (lines[i].empty()) continue;
        std::vector<std::string> f;
        size_t a = 0;
        for (;;) {
            const size_t c = lines[i].find(',', a);
            f.push_back(lines[i].substr(a, c == std::string::npos ? std::string::npos : c - a));
            if (c == std::string::npos) break;
            a = c + 1;
        }
        if (f.size() != 7) return fail(ABFS_EINVAL, "malformed trace row " + std::to_string(i));
        abfs_level_record r{};
        r.next_out_edges = ~0ull;   // not a trace-CSV column (unvisited: 0 = not recorded)
        r.level = std::strtoll(f[0].c_str(), nullptr, 10);
        r.kernel = r.variant = -1;
        for (int q = 0; q < 5; ++q)
            if (f[1] == kKernelNames[q]) r.kernel = q;
        for (int q = 0; q < 3; ++q)
            if (f[2] == kVariantNames[q]) r.variant = q;
        if (r.kernel < 0) return fail(ABFS_EINVAL, "'" + f[1] + "'");   // KeyError text
        if (r.variant < 0) return fail(ABFS_EINVAL, "'" + f[2] + "'");
        r.fallback = std::atoi(f[3].c_str()) != 0;
        r.frontier_size = std::strtoull(f[4].c_str(), nullptr, 10);
        r.elapsed_ns = std::strtoull(f[5].c_str(), nullptr, 10);
        r.prediction_ns = std::strtoull(f[6].c_str(), nullptr, 10);
        if (recs && cnt < cap) recs[cnt] = r;
        ++cnt;
    }
    *n = cnt;
    return ABFS_OK;
}
