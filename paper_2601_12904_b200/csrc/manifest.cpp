// FKVC manifest ("Manifest: JSON file mapping chunk_id -> relative
// path + variant + native_start"): a store's records saved as one FKVC file
// each plus a JSON index, and the index read back through the DISK -> GPU
// loader (store_load). The FKVC format carries no token ids, which the
// recompute gather needs, so every manifest entry also lists the chunk's
// tokens (an extension: readers of the spec's three fields ignore it).
//
//   {"format": "FKVC-manifest", "version": 1,
//    "records": [{"chunk_id": "<32 hex>", "path": "<32 hex>.fkvc",
//                 "variant": "ISOLATED" | "FUSED", "native_start": 9,
//                 "tokens": [17, 4, ...]}, ...]}
//
// Errors are FormatError kinds (common.hpp:33): unreadable file -> Io, JSON or
// schema violations and entries that disagree with their file's header ->
// Malformed; the FKVC reader's own kinds pass through.
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "engine.h"

namespace fragimpl {

namespace {

// ------------------------------------------------------------ minimal JSON
struct JVal {
  enum Kind { Null, Bool, Num, Str, Arr, Obj } kind = Null;
  bool b = false;
  double num = 0;
  std::string str;
  std::vector<JVal> arr;
  std::vector<std::pair<std::string, JVal>> obj;
  const JVal* get(const char* k) const {
    for (const auto& kv : obj)
      if (kv.first == k) return &kv.second;
    return nullptr;
  }
};

struct JParser {
  const char* p;
  const char* end;
  const char* path;
  [[noreturn]] void bad(const char* what) {
    fail_format(FRAG_FORMAT_MALFORMED, std::string("manifest JSON: ") + what + " (" + path + ")");
  }
  void ws() {
    while (p < end && (*p == ' ' || *p == '\n' || *p == '\r' || *p == '\t')) ++p;
  }
  bool lit(const char* s) {
    const size_t n = std::strlen(s);
    if ((size_t)(end - p) >= n && std::memcmp(p, s, n) == 0) {
      p += n;
      return true;
    }
    return false;
  }
  std::string string() {
    if (p >= end || *p != '"') bad("expected a string");
    ++p;
    std::string out;
    while (p < end && *p != '"') {
      char c = *p++;
      if (c == '\\') {
        if (p >= end) bad("unterminated escape");
        const char e = *p++;
        switch (e) {
          case '"': case '\\': case '/': out += e; break;
          case 'n': out += '\n'; break;
          case 't': out += '\t'; break;
          case 'r': out += '\r'; break;
          case 'b': out += '\b'; break;
          case 'f': out += '\f'; break;
          default: bad("unsupported escape");
        }
      } else {
        out += c;
      }
    }
    if (p >= end) bad("unterminated string");
    ++p;
    return out;
  }
  JVal value(int depth = 0) {
    if (depth > 16) bad("nesting too deep");
    ws();
    if (p >= end) bad("unexpected end");
    JVal v;
    if (*p == '{') {
      v.kind = JVal::Obj;
      ++p;
      ws();
      if (p < end && *p == '}') {
        ++p;
        return v;
      }
      for (;;) {
        ws();
        std::string k = string();
        ws();
        if (p >= end || *p != ':') bad("expected ':'");
        ++p;
        v.obj.emplace_back(std::move(k), value(depth + 1));
        ws();
        if (p < end && *p == ',') {
          ++p;
          continue;
        }
        if (p < end && *p == '}') {
          ++p;
          return v;
        }
        bad("expected ',' or '}'");
      }
    }
    if (*p == '[') {
      v.kind = JVal::Arr;
      ++p;
      ws();
      if (p < end && *p == ']') {
        ++p;
        return v;
      }
      for (;;) {
        v.arr.push_back(value(depth + 1));
        ws();
        if (p < end && *p == ',') {
          ++p;
          continue;
        }
        if (p < end && *p == ']') {
          ++p;
          return v;
        }
        bad("expected ',' or ']'");
      }
    }
    if (*p == '"') {
      v.kind = JVal::Str;
      v.str = string();
      return v;
    }
    if (lit("true")) {
      v.kind = JVal::Bool;
      v.b = true;
      return v;
    }
    if (lit("false")) {
      v.kind = JVal::Bool;
      return v;
    }
    if (lit("null")) return v;
    char* q = nullptr;
    const std::string num(p, (size_t)std::min<ptrdiff_t>(end - p, 64));
    v.num = std::strtod(num.c_str(), &q);
    if (q == num.c_str()) bad("unexpected character");
    p += q - num.c_str();
    v.kind = JVal::Num;
    return v;
  }
};

std::string read_text(const char* path) {
  FILE* f = std::fopen(path, "rb");
  if (!f) fail_format(FRAG_FORMAT_IO, std::string("cannot open manifest ") + path);
  std::string s;
  char buf[65536];
  size_t n;
  while ((n = std::fread(buf, 1, sizeof(buf), f)) > 0) s.append(buf, n);
  const bool err = std::ferror(f) != 0;
  std::fclose(f);
  if (err) fail_format(FRAG_FORMAT_IO, std::string("read error: ") + path);
  return s;
}

std::string hex_of(const frag_chunk_id& id) {
  static const char* d = "0123456789abcdef";
  std::string s(32, '0');
  for (int i = 0; i < 16; ++i) {
    s[2 * i] = d[id.bytes[i] >> 4];
    s[2 * i + 1] = d[id.bytes[i] & 15];
  }
  return s;
}

bool id_from_hex(const std::string& h, frag_chunk_id* id) {
  if (h.size() != 32) return false;
  auto nib = [](char c) -> int {
    if (c >= '0' && c <= '9') return c - '0';
    if (c >= 'a' && c <= 'f') return c - 'a' + 10;
    if (c >= 'A' && c <= 'F') return c - 'A' + 10;
    return -1;
  };
  for (int i = 0; i < 16; ++i) {
    const int a = nib(h[2 * i]), b = nib(h[2 * i + 1]);
    if (a < 0 || b < 0) return false;
    id->bytes[i] = (uint8_t)(a * 16 + b);
  }
  return true;
}

std::string dir_of(const std::string& path) {
  const size_t k = path.find_last_of('/');
  return k == std::string::npos ? std::string(".") : path.substr(0, k);
}

}  // namespace

std::vector<ManifestEntry> manifest_read(const char* path) {
  const std::string text = read_text(path);
  JParser jp{text.data(), text.data() + text.size(), path};
  const JVal root = jp.value();
  jp.ws();
  if (jp.p != jp.end) jp.bad("trailing data");
  auto bad = [&](const std::string& m) { fail_format(FRAG_FORMAT_MALFORMED, "manifest " + std::string(path) + ": " + m); };
  if (root.kind != JVal::Obj) bad("top level must be an object");
  const JVal* fmt = root.get("format");
  if (!fmt || fmt->kind != JVal::Str || fmt->str != "FKVC-manifest") bad("format must be \"FKVC-manifest\"");
  const JVal* ver = root.get("version");
  if (!ver || ver->kind != JVal::Num || ver->num != 1)
    fail_format(FRAG_FORMAT_BAD_VERSION, "manifest " + std::string(path) + ": version must be 1");
  const JVal* recs = root.get("records");
  if (!recs || recs->kind != JVal::Arr) bad("records must be an array");
  const std::string base = dir_of(path);
  std::vector<ManifestEntry> out;
  for (size_t i = 0; i < recs->arr.size(); ++i) {
    const JVal& r = recs->arr[i];
    const std::string at = "record " + std::to_string(i) + ": ";
    if (r.kind != JVal::Obj) bad(at + "not an object");
    ManifestEntry e;
    const JVal* cid = r.get("chunk_id");
    if (!cid || cid->kind != JVal::Str || !id_from_hex(cid->str, &e.id)) bad(at + "chunk_id must be 32 hex digits");
    const JVal* rel = r.get("path");
    if (!rel || rel->kind != JVal::Str || rel->str.empty()) bad(at + "path missing");
    e.path = rel->str[0] == '/' ? rel->str : base + "/" + rel->str;
    const JVal* var = r.get("variant");
    if (!var || var->kind != JVal::Str || (var->str != "ISOLATED" && var->str != "FUSED"))
      bad(at + "variant must be ISOLATED or FUSED");
    e.variant = var->str == "FUSED" ? FRAG_VARIANT_FUSED : FRAG_VARIANT_ISOLATED;
    const JVal* ns = r.get("native_start");
    if (!ns || ns->kind != JVal::Num || ns->num < 1 || ns->num != (double)(int32_t)ns->num)
      bad(at + "native_start must be an integer >= 1");
    e.native_start = (int32_t)ns->num;
    const JVal* tk = r.get("tokens");
    if (!tk || tk->kind != JVal::Arr || tk->arr.empty()) bad(at + "tokens must be a non-empty array");
    for (const JVal& t : tk->arr) {
      if (t.kind != JVal::Num || t.num < 0 || t.num != (double)(int32_t)t.num) bad(at + "token ids must be integers");
      e.tokens.push_back((int32_t)t.num);
    }
    // the entry must agree with its file's header (FKVC reader kinds pass through)
    frag_fkvc_header h{};
    fkvc_read(e.path.c_str(), &h, nullptr, nullptr, 0);
    if (std::memcmp(h.id.bytes, e.id.bytes, 16) != 0) bad(at + "chunk_id differs from the file's");
    if (h.variant != e.variant || h.native_start != e.native_start) bad(at + "variant / native_start differ from the file's");
    if (h.tokens != (int32_t)e.tokens.size()) bad(at + "token count differs from the file's");
    out.push_back(std::move(e));
  }
  return out;
}

int manifest_save(Store* st, const char* dir, const char* name) {
  struct Item {
    frag_chunk_id id;
    int variant, native_start;
    std::vector<int32_t> tok;
  };
  std::vector<Item> items;
  {
    std::shared_lock<std::shared_mutex> g(st->mu);
    for (const auto& kv : st->recs) {
      const Record* r = kv.second.get();
      if (r->tier == FRAG_TIER_PEER) continue;  // another GPU's record: its owner saves it
      items.push_back(Item{r->id, r->variant, r->native_start, r->tok_host});
    }
  }
  // deterministic order (by chunk id)
  std::sort(items.begin(), items.end(),
            [](const Item& a, const Item& b) { return std::memcmp(a.id.bytes, b.id.bytes, 16) < 0; });
  std::string js = "{\"format\": \"FKVC-manifest\", \"version\": 1, \"records\": [";
  for (size_t i = 0; i < items.size(); ++i) {
    const Item& it = items[i];
    const std::string hx = hex_of(it.id);
    const std::string file = hx + ".fkvc";
    store_save(st, it.id, (std::string(dir) + "/" + file).c_str());
    js += i ? ",\n  " : "\n  ";
    js += "{\"chunk_id\": \"" + hx + "\", \"path\": \"" + file + "\", \"variant\": \"" +
          (it.variant == FRAG_VARIANT_FUSED ? "FUSED" : "ISOLATED") +
          "\", \"native_start\": " + std::to_string(it.native_start) + ", \"tokens\": [";
    for (size_t t = 0; t < it.tok.size(); ++t) {
      if (t) js += ", ";
      js += std::to_string(it.tok[t]);
    }
    js += "]}";
  }
  js += "\n]}\n";
  const std::string mpath = std::string(dir) + "/" + (name && *name ? name : "manifest.json");
  FILE* f = std::fopen(mpath.c_str(), "wb");
  if (!f) fail_format(FRAG_FORMAT_IO, "cannot create " + mpath);
  const bool ok = std::fwrite(js.data(), 1, js.size(), f) == js.size();
  if (std::fclose(f) != 0 || !ok) fail_format(FRAG_FORMAT_IO, "write failed: " + mpath);
  return (int)items.size();
}

int manifest_load(Store* st, const char* path, bool overwrite, cudaStream_t s) {
  const std::vector<ManifestEntry> es = manifest_read(path);  // validated before anything is inserted
  for (const ManifestEntry& e : es) {
    frag_chunk_id got;
    store_load(st, e.path.c_str(), e.tokens.data(), (int)e.tokens.size(), overwrite, s, &got);
  }
  return (int)es.size();
}

}  // namespace fragimpl
