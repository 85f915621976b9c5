// tuning_cache.cpp — the persisted scheduler decisions (the reference's
// tuning cache, /root/reference/proj/include/deepfusion/tuner.hpp:91-113).
//
// What is kept from the reference is the contract: one human-readable JSON
// document {"format_version": 1, "entries": [ScheduleEntry...]}, one entry
// per (shape.batch, shape.d_model, shape.d_ff, fingerprint), store = insert
// or replace, lookup of an absent file or key = miss, an unparsable file or
// a different format_version = CacheError (DFK_ERR_CACHE), safe under
// concurrent writers and readers (threads and processes).
//
// The mechanism is this library's own:
//   * a store is a read-merge-publish transaction serialised by a process
//     mutex plus flock() on a sidecar "<path>.lock" (never on the document
//     itself), and the new document is published by writing a private
//     temporary file in the same directory and rename()-ing it over <path>;
//   * a lookup therefore needs no lock at all: rename is atomic, so a
//     reader opens either the previous document or the new one, never a
//     partially written file.
#include <fcntl.h>
#include <sys/file.h>
#include <sys/stat.h>
#include <unistd.h>

#include <atomic>
#include <cerrno>
#include <cstdio>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <mutex>
#include <sstream>
#include <string>

#include <json.hpp>

#include "internal.h"

using namespace dfk;
using nlohmann::json;

namespace {

constexpr int kSchemaVersion = 1;  // tuner.hpp:93 kCacheFormatVersion

struct CacheFailure {
  std::string what;
};

// Whole file as a string; false when it does not exist.
bool slurp(const std::string& path, std::string* text) {
  std::ifstream in(path, std::ios::binary);
  if (!in) return false;
  std::ostringstream ss;
  ss << in.rdbuf();
  *text = ss.str();
  return true;
}

// The parsed document, or an empty document for an absent / empty file.
json load_document(const std::string& path) {
  std::string text;
  if (!slurp(path, &text) || text.empty())
    return json{{"format_version", kSchemaVersion}, {"entries", json::array()}};
  json doc = json::parse(text, nullptr, /*allow_exceptions=*/false);
  if (doc.is_discarded() || !doc.is_object())
    throw CacheFailure{"tuning cache " + path + ": not a valid JSON document (corrupt file)"};
  auto v = doc.find("format_version");
  if (v == doc.end() || !v->is_number_integer())
    throw CacheFailure{"tuning cache " + path + ": no integer format_version field"};
  if (v->get<int>() != kSchemaVersion)
    throw CacheFailure{"tuning cache " + path + ": written with schema version " +
                       std::to_string(v->get<int>()) + ", this library understands version " +
                       std::to_string(kSchemaVersion)};
  auto e = doc.find("entries");
  if (e == doc.end() || !e->is_array())
    throw CacheFailure{"tuning cache " + path + ": no entries array"};
  return doc;
}

// (batch, d_model, d_ff, fingerprint) of one entry; throws on a malformed one.
struct Key {
  int64_t b, dm, df;
  std::string fp;
  bool operator==(const Key& o) const {
    return b == o.b && dm == o.dm && df == o.df && fp == o.fp;
  }
};

Key key_of(const json& entry, const std::string& path) {
  auto bad = [&](const char* what) {
    return CacheFailure{"tuning cache " + path + ": entry " + what};
  };
  if (!entry.is_object()) throw bad("is not an object");
  auto s = entry.find("shape");
  auto f = entry.find("fingerprint");
  if (s == entry.end() || !s->is_object()) throw bad("has no shape object");
  if (f == entry.end() || !f->is_string()) throw bad("has no fingerprint string");
  Key k;
  for (auto [name, dst] : {std::pair<const char*, int64_t*>{"batch", &k.b},
                           {"d_model", &k.dm}, {"d_ff", &k.df}}) {
    auto it = s->find(name);
    if (it == s->end() || !it->is_number_integer()) throw bad("has a malformed shape");
    *dst = it->get<int64_t>();
  }
  k.fp = f->get<std::string>();
  return k;
}

std::mutex& writers_mutex() {
  static std::mutex m;
  return m;
}

// Exclusive advisory lock on <path>.lock for the duration of one store.
class SidecarLock {
 public:
  explicit SidecarLock(const std::string& path) {
    fd_ = ::open((path + ".lock").c_str(), O_RDWR | O_CREAT | O_CLOEXEC, 0644);
    if (fd_ < 0)
      throw CacheFailure{"tuning cache " + path + ": cannot create lock file (" +
                         std::strerror(errno) + ")"};
    while (::flock(fd_, LOCK_EX) != 0 && errno == EINTR) {
    }
  }
  ~SidecarLock() {
    if (fd_ >= 0) ::close(fd_);  // closing the descriptor drops the lock
  }
  SidecarLock(const SidecarLock&) = delete;
  SidecarLock& operator=(const SidecarLock&) = delete;

 private:
  int fd_ = -1;
};

// Writes `text` to a private file next to `path`, then renames it over it.
void publish(const std::string& path, const std::string& text) {
  static std::atomic<unsigned> serial{0};
  const std::string tmp = path + ".tmp-" + std::to_string(::getpid()) + "-" +
                          std::to_string(serial.fetch_add(1));
  const int fd = ::open(tmp.c_str(), O_WRONLY | O_CREAT | O_TRUNC | O_CLOEXEC, 0644);
  if (fd < 0)
    throw CacheFailure{"tuning cache " + path + ": cannot write (" + std::strerror(errno) +
                       ")"};
  size_t off = 0;
  while (off < text.size()) {
    const ssize_t n = ::write(fd, text.data() + off, text.size() - off);
    if (n < 0 && errno == EINTR) continue;
    if (n <= 0) {
      ::close(fd);
      ::unlink(tmp.c_str());
      throw CacheFailure{"tuning cache " + path + ": short write"};
    }
    off += static_cast<size_t>(n);
  }
  ::fsync(fd);
  ::close(fd);
  if (::rename(tmp.c_str(), path.c_str()) != 0) {
    const std::string why = std::strerror(errno);
    ::unlink(tmp.c_str());
    throw CacheFailure{"tuning cache " + path + ": cannot replace (" + why + ")"};
  }
}

}  // namespace

namespace dfk {

// Lookup: true and *hit = the entry when (B, dm, df, fp) is present.
bool cache_find(const std::string& path, int64_t B, int64_t dm, int64_t df,
                const std::string& fp, std::string* hit, std::string* err) {
  try {
    const json doc = load_document(path);
    const Key want{B, dm, df, fp};
    for (const json& e : doc["entries"]) {
      if (key_of(e, path) == want) {
        *hit = e.dump();
        return true;
      }
    }
    return false;
  } catch (const CacheFailure& f) {
    *err = f.what;
    return false;
  }
}

// Insert-or-replace of one serialised entry; "" on success, else the error.
std::string cache_put(const std::string& path, const std::string& entry_text) {
  try {
    json entry = json::parse(entry_text, nullptr, false);
    if (entry.is_discarded())
      throw CacheFailure{"tuning cache " + path + ": the new entry is not valid JSON"};
    const Key k = key_of(entry, path);
    std::filesystem::path p(path);
    if (p.has_parent_path()) {
      std::error_code ec;
      std::filesystem::create_directories(p.parent_path(), ec);
    }
    std::lock_guard<std::mutex> in_process(writers_mutex());
    SidecarLock across_processes(path);
    json doc = load_document(path);
    json& entries = doc["entries"];
    bool replaced = false;
    for (json& e : entries) {
      if (key_of(e, path) == k) {
        e = entry;
        replaced = true;
        break;
      }
    }
    if (!replaced) entries.push_back(std::move(entry));
    publish(path, doc.dump(2) + "\n");
    return "";
  } catch (const CacheFailure& f) {
    return f.what;
  }
}

}  // namespace dfk

extern "C" {

int dfk_cache_lookup(const char* path, int64_t batch, int64_t d_model, int64_t d_ff,
                     const char* fingerprint, char* entry_json, size_t len,
                     size_t* needed, int32_t* found) {
  if (!path || !fingerprint || !found) return fail(DFK_ERR_INVALID, "null argument");
  *found = 0;
  if (needed) *needed = 0;
  std::string hit, err;
  if (!cache_find(path, batch, d_model, d_ff, fingerprint, &hit, &err)) {
    if (!err.empty()) return fail(DFK_ERR_CACHE, err);
    return DFK_OK;
  }
  *found = 1;
  if (needed) *needed = hit.size() + 1;
  if (entry_json) {
    if (len < hit.size() + 1)
      return fail(DFK_ERR_INVALID, "entry buffer too small (need " +
                                       std::to_string(hit.size() + 1) + " bytes)");
    std::memcpy(entry_json, hit.c_str(), hit.size() + 1);
  }
  return DFK_OK;
}

int dfk_cache_store(const char* path, const char* entry_json) {
  if (!path || !entry_json) return fail(DFK_ERR_INVALID, "null argument");
  if (!*path) return fail(DFK_ERR_INVALID, "empty cache path");
  const std::string err = cache_put(path, entry_json);
  if (!err.empty()) return fail(DFK_ERR_CACHE, err);
  return DFK_OK;
}

}  // extern "C"
