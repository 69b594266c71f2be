// Native, multi-threaded host tokenizer feeding the packed varlen batch (SURVEY.md §8(f)
// row 4; the paper's C++ multi-threaded tokenizer).  Host code only.
//
// Semantics are the Python restatement's (paper_2209_09130_b200/tokenization.py, itself
// pinned to the reference's tests and calibration goldens) for every input that is pure
// ASCII: NFC/NFD are the identity on ASCII, the Cc controls other than \t\n\r are dropped,
// \t\n\r become spaces, optional lower-casing, whitespace split with ASCII punctuation
// isolated (char_mode: every character a word), greedy longest-match-first wordpiece with
// "##" continuations, [UNK] for words over 100 characters or without a match, then
// [CLS] a [SEP] (b [SEP]) with longest-first truncation and padding to max_seq_len.
// Inputs containing any non-ASCII byte are not tokenized here: they are flagged and the
// caller runs the Python path for them (Unicode normalisation / categories), so results
// are identical for every input.
#include <condition_variable>
#include <cstdint>
#include <cstring>
#include <functional>
#include <mutex>
#include <string>
#include <string_view>
#include <thread>
#include <unordered_map>
#include <vector>

namespace {

// Persistent workers (thread creation costs ~50-300 us, more than a small batch's work)
class Pool {
 public:
  ~Pool() {
    {
      std::lock_guard<std::mutex> g(m_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto& t : threads_) t.join();
  }
  // run fn(tid) for tid in [0, n) on n-1 workers + the caller; returns when all are done
  void run(int n, const std::function<void(int)>& fn) {
    std::lock_guard<std::mutex> call(call_);   // one batch at a time per tokenizer
    while (int(threads_.size()) < n - 1) {
      const int id = int(threads_.size()) + 1;
      threads_.emplace_back([this, id] { loop(id); });
    }
    {
      std::lock_guard<std::mutex> g(m_);
      fn_ = &fn;
      active_ = n;
      pending_ = n - 1;
      ++gen_;
    }
    cv_.notify_all();
    fn(0);
    std::unique_lock<std::mutex> g(m_);
    done_.wait(g, [this] { return pending_ == 0; });
    fn_ = nullptr;
  }

 private:
  void loop(int id) {
    unsigned long seen = 0;
    for (;;) {
      const std::function<void(int)>* fn;
      {
        std::unique_lock<std::mutex> g(m_);
        cv_.wait(g, [&] { return stop_ || gen_ != seen; });
        if (stop_) return;
        seen = gen_;
        if (id >= active_) continue;
        fn = fn_;
      }
      (*fn)(id);
      {
        std::lock_guard<std::mutex> g(m_);
        if (--pending_ == 0) done_.notify_one();
      }
    }
  }
  std::vector<std::thread> threads_;
  std::mutex m_, call_;
  std::condition_variable cv_, done_;
  const std::function<void(int)>* fn_ = nullptr;
  int active_ = 0, pending_ = 0;
  unsigned long gen_ = 0;
  bool stop_ = false;
};

struct Tokenizer {
  std::unordered_map<std::string, int> ids;
  bool lower = true, char_mode = false;
  int max_len = 128;
  int cls = 0, sep = 0, pad = 0, unk = 0;
  Pool pool;
};

bool ascii_only(const char* s) {
  for (; *s; ++s)
    if (static_cast<unsigned char>(*s) >= 0x80) return false;
  return true;
}

bool is_punct(unsigned char c) {
  return (c >= 33 && c <= 47) || (c >= 58 && c <= 64) || (c >= 91 && c <= 96) || (c >= 123 && c <= 126);
}

// tokenization._normalize + _basic_words on ASCII text
void basic_words(const Tokenizer& t, const char* text, std::vector<std::string>& words) {
  words.clear();
  std::string cur;
  auto flush = [&]() {
    if (!cur.empty()) {
      words.push_back(cur);
      cur.clear();
    }
  };
  for (const char* p = text; *p; ++p) {
    unsigned char c = static_cast<unsigned char>(*p);
    if (c == '\t' || c == '\n' || c == '\r') c = ' ';
    else if (c < 0x20 || c == 0x7f) continue;        // Cc controls (and \x00) are dropped
    if (t.lower && c >= 'A' && c <= 'Z') c = static_cast<unsigned char>(c - 'A' + 'a');
    if (c == ' ') {
      flush();
    } else if (t.char_mode || is_punct(c)) {
      flush();
      words.emplace_back(1, static_cast<char>(c));
    } else {
      cur.push_back(static_cast<char>(c));
    }
  }
  flush();
}

// tokenization.wordpiece
void wordpiece(const Tokenizer& t, const std::string& w, std::vector<int>& out, std::string& scratch) {
  if (w.size() > 100) {
    out.push_back(t.unk);
    return;
  }
  const size_t start = out.size();
  size_t pos = 0;
  while (pos < w.size()) {
    int match = -1;
    size_t end = w.size();
    for (; end > pos; --end) {
      scratch.clear();
      if (pos > 0) scratch.append("##");
      scratch.append(w, pos, end - pos);
      auto it = t.ids.find(scratch);
      if (it != t.ids.end()) {
        match = it->second;
        break;
      }
    }
    if (match < 0) {
      out.resize(start);
      out.push_back(t.unk);
      return;
    }
    out.push_back(match);
    pos = end;
  }
}

void tokenize(const Tokenizer& t, const char* text, std::vector<int>& out, std::vector<std::string>& words,
              std::string& scratch) {
  out.clear();
  basic_words(t, text, words);
  for (const auto& w : words) wordpiece(t, w, out, scratch);
}

// tokenization.encode
void encode(const Tokenizer& t, const char* a_text, const char* b_text, int32_t* ids, int32_t* segs, int32_t* att,
            std::vector<int>& a, std::vector<int>& b, std::vector<std::string>& words, std::string& scratch) {
  const int limit = t.max_len;
  tokenize(t, a_text, a, words, scratch);
  int n = 0;
  if (!b_text) {
    if (int(a.size()) > std::max(limit - 2, 0)) a.resize(std::max(limit - 2, 0));
    ids[n] = t.cls; segs[n++] = 0;
    for (int v : a) { ids[n] = v; segs[n++] = 0; }
    ids[n] = t.sep; segs[n++] = 0;
  } else {
    tokenize(t, b_text, b, words, scratch);
    const size_t budget = size_t(std::max(limit - 3, 0));
    while (a.size() + b.size() > budget) {
      if (a.size() > b.size()) a.pop_back();
      else b.pop_back();
    }
    ids[n] = t.cls; segs[n++] = 0;
    for (int v : a) { ids[n] = v; segs[n++] = 0; }
    ids[n] = t.sep; segs[n++] = 0;
    for (int v : b) { ids[n] = v; segs[n++] = 1; }
    ids[n] = t.sep; segs[n++] = 1;
  }
  *att = n;
  const int32_t pad_seg = b_text ? segs[n - 1] : 0;
  for (int k = n; k < limit; ++k) {
    ids[k] = t.pad;
    segs[k] = pad_seg;
  }
}

}  // namespace

extern "C" {

struct samp_tokenizer;

// tokens[i] is the token of id i (UTF-8); the special tokens must be present (the Python
// Vocab validates the same and raises ConfigurationError first)
samp_tokenizer* samp_tokenizer_create(const char* const* tokens, int ntokens, int do_lower_case, int max_seq_len,
                                      int char_mode) {
  auto* t = new Tokenizer();
  t->ids.reserve(size_t(ntokens) * 2);
  for (int i = 0; i < ntokens; ++i) t->ids.emplace(tokens[i], i);
  t->lower = do_lower_case != 0;
  t->char_mode = char_mode != 0;
  t->max_len = max_seq_len;
  auto get = [&](const char* s) {
    auto it = t->ids.find(s);
    return it == t->ids.end() ? -1 : it->second;
  };
  t->cls = get("[CLS]");
  t->sep = get("[SEP]");
  t->pad = get("[PAD]");
  t->unk = get("[UNK]");
  if (t->cls < 0 || t->sep < 0 || t->pad < 0 || t->unk < 0 || max_seq_len < 3) {
    delete t;
    return nullptr;
  }
  return reinterpret_cast<samp_tokenizer*>(t);
}

void samp_tokenizer_destroy(samp_tokenizer* h) { delete reinterpret_cast<Tokenizer*>(h); }

// Encode n items (text_b may be null, or hold null entries for single texts) into padded
// rows ids/segs [n][max_seq_len] and att[n], on nthreads host threads.  Items with any
// non-ASCII byte get fallback[i] = 1 and untouched rows (the caller encodes them).
// Returns the number of fallback items.
int samp_tokenize_batch(samp_tokenizer* h, const char* const* text_a, const char* const* text_b, int n, int nthreads,
                        int32_t* ids, int32_t* segs, int32_t* att, uint8_t* fallback) {
  const Tokenizer& t = *reinterpret_cast<Tokenizer*>(h);
  const int L = t.max_len;
  // a worker per >= 8 texts (a 128-token text is ~10 us of work)
  nthreads = std::max(1, std::min(nthreads, (n + 7) / 8));
  std::vector<int> nfb(nthreads, 0);
  auto work = [&](int tid) {
    std::vector<int> a, b;
    std::vector<std::string> words;
    std::string scratch;
    for (int i = tid; i < n; i += nthreads) {
      const char* bt = text_b ? text_b[i] : nullptr;
      if (!ascii_only(text_a[i]) || (bt && !ascii_only(bt))) {
        fallback[i] = 1;
        ++nfb[tid];
        continue;
      }
      fallback[i] = 0;
      encode(t, text_a[i], bt, ids + size_t(i) * L, segs + size_t(i) * L, att + i, a, b, words, scratch);
    }
  };
  if (nthreads == 1) {
    work(0);
  } else {
    reinterpret_cast<Tokenizer*>(h)->pool.run(nthreads, work);
  }
  int total = 0;
  for (int v : nfb) total += v;
  return total;
}

}  // extern "C"
